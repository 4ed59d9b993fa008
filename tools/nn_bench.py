"""Time one streaming kernel shape in isolation (CUDA events, warm, back to back):
  python tools/nn_bench.py nn M K C   -> Y = X M  (X M x K, no norms: the alpha pass)
  python tools/nn_bench.py tn M N L   -> Z = X^T Y (the beta pass)
  python tools/nn_bench.py gram M W [LD] -> X^T X over the first W of LD columns
Prints ms and TFLOP/s (algorithmic flops)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1612_08709_b200 as tk  # noqa: E402

kind = sys.argv[1]
a, b, c = (int(x) for x in sys.argv[2:5])
ld = int(sys.argv[5]) if len(sys.argv) > 5 else None
g = torch.Generator(device="cuda").manual_seed(0)
f = torch.float64
if kind == "nn":
    X = torch.randn(a, max(ld or 0, b + (b & 1)), device="cuda", dtype=f, generator=g)[:, :b]
    M = torch.randn(b, c, device="cuda", dtype=f, generator=g)
    norms = os.environ.get("NORMS") == "1"
    fn = lambda: tk.matmul(X, M, norms=norms)  # noqa: E731
    flops = 2.0 * a * b * c
elif kind == "tn":
    X = torch.randn(a, b, device="cuda", dtype=f, generator=g)
    Y = torch.randn(a, c + (c & 1), device="cuda", dtype=f, generator=g)
    fn = lambda: tk.matmul_tn(X, Y, c)  # noqa: E731
    flops = 2.0 * a * b * c
else:  # gram M W LD
    X = torch.randn(a, max(c, b), device="cuda", dtype=f, generator=g)[:, :b]
    fn = lambda: tk.gram(X)  # noqa: E731
    flops = 1.0 * a * b * (b + 1)
for _ in range(3):
    fn()
torch.cuda.synchronize()
reps = 10
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    fn()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"{kind} {a}x{b}x{c} env={ {k: v for k, v in os.environ.items() if k.startswith('TSSVD_')} } ms={ms:.3f} TF={flops / ms / 1e9:.2f}",
      flush=True)
