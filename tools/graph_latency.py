"""Per-call device time of lowrank_svd with and without the per-call CUDA graph (TSSVD_GRAPH),
on small shapes where launch latency matters and on c3."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1612_08709_b200 as tk  # noqa: E402
import synth  # noqa: E402

for name, m, n in [("c3", 4_000, 1_000), ("c3", 50_000, 5_000), ("c3", None, None)]:
    d = synth.config_inputs(name, m=m, n=n)
    A = torch.from_numpy(d["A"]).cuda()
    Om = torch.from_numpy(d["Omega"]).cuda()
    for _ in range(3):
        tk.lowrank_svd(A, Om, d["iters"], d["k"])
    torch.cuda.synchronize()
    reps = 20 if m else 5
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        tk.lowrank_svd(A, Om, d["iters"], d["k"])
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} {A.shape[0]}x{A.shape[1]} graph={os.environ.get('TSSVD_GRAPH', '1')}: device "
          f"{e0.elapsed_time(e1) / reps:.3f} ms/call, host {1e3 * (time.perf_counter() - t0) / reps:.3f} ms/call, "
          f"launches {tk.last_stats()['kernel_launches']}", flush=True)
    del A
