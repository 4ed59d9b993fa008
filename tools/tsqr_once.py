"""One tsqr_svd call (Alg. 1 or 2) on an m x n Gaussian matrix (ncu launch lists)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1612_08709_b200 as tk  # noqa: E402
import synth  # noqa: E402

m, n, passes = (int(x) for x in (sys.argv[1:] + ["2000000", "100", "1"])[:3])
dev = torch.device("cuda", 0)
A = torch.randn((m, n), dtype=torch.float64, device=dev)
ph, pm = synth.mixing_params(n, 1)
tk.tsqr_svd(A, torch.from_numpy(ph).to(dev), torch.from_numpy(pm).to(dev), passes=passes)
torch.cuda.synchronize()
