"""Wide eigensolver (n > 256) on the paper's n = 2000 Gram (Eq. originalmat + testS, m = 10,000) and
on random Grams: eigenvalues vs LAPACK, residual, orthonormality of the kept vectors, time."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1612_08709_b200 as tk  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
cases = []
a, s = synth.paper_test_matrix(10_000, 2_000)
cases.append(("paper n=2000", a.T @ a))
for n in (300, 1000, 2000):
    x = np.random.default_rng(n).standard_normal((3 * n, n))
    cases.append((f"random n={n}", x.T @ x))
for name, b in cases:
    B = torch.from_numpy(b).to(dev)
    tk.sym_eig(B)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lam, v, sw = tk.sym_eig(B)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    lam, v = lam.cpu().numpy(), v.cpu().numpy()
    d = np.sort(np.linalg.eigvalsh(b))[::-1]
    K = int(np.sum(lam > 0))
    vk = v[:, :K]
    print(f"{name}: {dt * 1e3:.1f} ms, sweeps {sw}, K {K}, max|dlam|/lam1 {np.max(np.abs(lam - np.maximum(d, 0))) / d[0]:.2e}, "
          f"ortho {np.max(np.abs(vk.T @ vk - np.eye(K))):.2e}, resid {np.max(np.abs(b @ vk - vk * lam[:K])) / d[0]:.2e}",
          flush=True)
