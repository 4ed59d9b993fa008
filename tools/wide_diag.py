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
        vt = synth.dct_columns(2_000, 2_000)  # exact right singular vectors (Eq. originalmat)
        resid_g = np.max(np.abs(a @ vg - ug * sg)) if passes else 0
        resid_r = np.max(np.abs(a @ vr - ur * sr))
        print("  max|A V - U S|: gpu", resid_g, "oracle", resid_r, flush=True)
        j, wg, wr = 0, 0.0, 0.0
        while j < sr.size:
            e = j + 1
            while e < sr.size and abs(sr[e] - sr[j]) <= 1e-8:
                e += 1
            wg = max(wg, np.linalg.norm(vg[:, j:e] - vt[:, j:e] @ (vt[:, j:e].T @ vg[:, j:e]), 2))
            wr = max(wr, np.linalg.norm(vr[:, j:e] - vt[:, j:e] @ (vt[:, j:e].T @ vr[:, j:e]), 2))
            j = e
        print("  max sine to the TRUE right subspaces: gpu", wg, "oracle", wr, flush=True)
        j = 0
        while j < sr.size:
            e = j + 1
            while e < sr.size and abs(sr[e] - sr[j]) <= 1e-8:
                e += 1
            su = np.linalg.norm(ug[:, j:e] - ur[:, j:e] @ (ur[:, j:e].T @ ug[:, j:e]), 2)
            sv = np.linalg.norm(vg[:, j:e] - vr[:, j:e] @ (vr[:, j:e].T @ vg[:, j:e]), 2)
            if max(su, sv) > 1e-10:
                print(f"  group [{j},{e}) sigma {sr[j]:.6f} sine U {su:.2e} V {sv:.2e}", flush=True)
            j = e
