"""Small workloads that exercise every kernel of the library, for compute-sanitizer:
  compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize_run.py
tssvd at c1 (narrow: device-side decisions), reduced c2 (host decisions, warp-block Jacobi),
reduced c4 (w = 200: the 4-CTA cluster eigensolver with the st.async DSMEM exchange and the
cluster SVD), lowrank at reduced c3 (Alg. 8), a stream-K matmul and a split matmul_tn."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1612_08709_b200 as tk  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
for name, m in [("c1", None), ("c2", 20_000), ("c4", 20_000)]:
    d = synth.config_inputs(name, m=m)
    u, s, v = tk.tssvd(torch.from_numpy(d["A"]).to(dev))
    print(name, "rank", s.numel(), tk.last_stats()["jacobi_sweeps"], flush=True)
d = synth.config_inputs("c3", m=3_000, n=600)
u, s, v = tk.lowrank_svd(torch.from_numpy(d["A"]).to(dev), torch.from_numpy(d["Omega"]).to(dev), 1, 10)
print("lowrank rank", s.numel(), flush=True)
X = torch.randn(1_000, 4_000, dtype=torch.float64, device=dev)
y = tk.matmul(X, torch.randn(4_000, 25, dtype=torch.float64, device=dev))
z = tk.matmul_tn(X, torch.randn(1_000, 26, dtype=torch.float64, device=dev), 25)
torch.cuda.synchronize()
print("ok", flush=True)
