"""Diagnostics of the wide core on the paper's n = 2000 matrices: per-group subspace sines vs the
oracle, orthonormality of U and V, for Alg. 3 and Alg. 4."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1612_08709_b200 as tk  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
for name, (a, sig), wp in [("staircase", synth.paper_staircase_matrix(10_000, 2_000), 1e-11),
                           ("table5", synth.paper_test_matrix(10_000, 2_000), 1e-12)]:
    for passes in (1, 2):
        u, s, v = tk.tssvd(torch.from_numpy(a).to(dev), wp=wp, passes=passes)
        st = tk.last_stats()
        ug, sg, vg = u.cpu().numpy(), s.cpu().numpy(), v.cpu().numpy()
        ur, sr, vr = oracle.tssvd(a, wp, passes)
        print(name, passes, "rank", sg.size, sr.size, "sweeps", st["jacobi_sweeps"], "ortho U/V",
              oracle.ortho_error(ug), oracle.ortho_error(vg), "ref", oracle.ortho_error(ur), oracle.ortho_error(vr),
              "dsig", np.max(np.abs(sg - sr)) if sg.size == sr.size else None, flush=True)
        if sg.size != sr.size or name != "staircase":
            continue
        j = 0
        while j < sr.size:
            e = j + 1
            while e < sr.size and abs(sr[e] - sr[j]) <= 1e-8:
                e += 1
            su = np.sqrt(max(0, 1 - np.min(np.linalg.svd(ug[:, j:e].T @ ur[:, j:e], compute_uv=False)) ** 2))
            sv = np.sqrt(max(0, 1 - np.min(np.linalg.svd(vg[:, j:e].T @ vr[:, j:e], compute_uv=False)) ** 2))
            if max(su, sv) > 1e-10:
                print(f"  group [{j},{e}) sigma {sr[j]:.6f} sine U {su:.2e} V {sv:.2e}", flush=True)
            j = e
