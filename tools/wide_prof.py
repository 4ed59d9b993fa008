"""Phase split of the wide block-Jacobi sweeps (CTA 0's clock64 marks; needs a library built with
-D WIDE_PROF, loaded through TSSVD_LIB).  Phases: partial Gram, grid sync 1, sum+test,
inner sweep, apply, grid sync 2 -- cycles per outer round."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1612_08709_b200 as tk  # noqa: E402
from paper_1612_08709_b200 import _lib  # noqa: E402

lib = _lib.lib()
for n in (300, 1000, 2000):
    x = np.random.default_rng(n).standard_normal((3 * n, n))
    B = torch.from_numpy(x.T @ x).cuda()
    tk.sym_eig(B)
    buf = (ctypes.c_ulonglong * 8)()
    lib.tssvd_wide_prof(buf)
    lam, v, sw = tk.sym_eig(B)
    torch.cuda.synchronize()
    lib.tssvd_wide_prof(buf)
    nb = ((n + 31) // 32 * 32) // 16
    rounds = sw * (nb - 1)
    names = ["gram", "sync1", "sum+test", "inner", "apply", "sync2"]
    print(f"n={n} S={os.environ.get('TSSVD_WIDE_S', 'auto')} sweeps {sw} rounds {rounds}: " +
          ", ".join(f"{nm} {buf[i] / rounds:.0f}" for i, nm in enumerate(names)) + " cycles/round", flush=True)
