"""One tridiagonal-QL solve of a c2-like second-pass Gram (n = 55) and one of n = 92, for ncu."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import paper_1612_08709_b200 as tk  # noqa: E402
from test_gpu_ql import second_pass_gram  # noqa: E402

for m, n in ((20_000, 100), (40_000, 200)):
    z = torch.from_numpy(second_pass_gram(m, n)).cuda()
    for _ in range(3):
        lam, v, it = tk.sym_eig_ql(z)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        tk.sym_eig_ql(z)
    e1.record()
    torch.cuda.synchronize()
    ql = e0.elapsed_time(e1) / 10
    e0.record()
    for _ in range(10):
        tk.sym_eig(z)
    e1.record()
    torch.cuda.synchronize()
    print(f"n={z.shape[0]} QL iterations {it}: {ql:.3f} ms per call (incl. copy + sync); "
          f"Jacobi {e0.elapsed_time(e1) / 10:.3f} ms", flush=True)
