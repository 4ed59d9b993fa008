"""Accuracy of the wide Gram (gemm_tn block columns) vs numpy, and of the wide tssvd's U
orthonormality on the staircase under rotation-threshold scalings (TSSVD_WIDE_TOL)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1612_08709_b200 as tk  # noqa: E402
import synth  # noqa: E402

a, s = synth.paper_staircase_matrix(10_000, 2_000)
A = torch.from_numpy(a).cuda()
g = torch.empty(2000, 2000, dtype=torch.float64)
for j0 in range(0, 2000, 128):
    l = min(128, 2000 - j0)
    g[j0:, j0:j0 + l] = tk.matmul_tn(A[:, j0:], A[:, j0:j0 + l].contiguous(), l).cpu()
g = torch.tril(g) + torch.tril(g, -1).T
b = a.T @ a
exact = (synth.dct_columns(2000, 2000) * s ** 2) @ synth.dct_columns(2000, 2000).T
print("gram: max|G_gpu - G_np|", np.max(np.abs(g.numpy() - b)), "vs exact: gpu", np.max(np.abs(g.numpy() - exact)),
      "np", np.max(np.abs(b - exact)), flush=True)
for passes in (1, 2):
    u, sg, v = tk.tssvd(A, wp=1e-11, passes=passes)
    st = tk.last_stats()
    print(os.environ.get("TSSVD_WIDE_TOL", "1"), passes, "sweeps", st["jacobi_sweeps"], "ortho U", oracle.ortho_error(u.cpu().numpy()),
          "V", oracle.ortho_error(v.cpu().numpy()), flush=True)
