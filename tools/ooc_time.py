"""Out-of-core lowrank_svd (opts.host_io = 2) at c3's full size: A (32 GB) stays in pinned host memory and
each of the 6 passes streams it over PCIe.  Prints the call time, the effective host->device stream rate
and the in-core (host_io = 1) call for comparison."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1612_08709_b200 as tk  # noqa: E402
import synth  # noqa: E402

d = synth.config_inputs("c3")
a = torch.from_numpy(d["A"]).pin_memory()
om = torch.from_numpy(d["Omega"]).pin_memory()
for ooc in (True, False):
    tk.lowrank_svd(a, om, d["iters"], d["k"], out_of_core=ooc)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    u, s, v = tk.lowrank_svd(a, om, d["iters"], d["k"], out_of_core=ooc)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    passes = 2 * d["iters"] + 2
    print(f"out_of_core={ooc}: {dt * 1e3:.1f} ms per call, A streamed {passes if ooc else 1} x {a.numel() * 8 / 1e9:.1f} GB "
          f"-> {(passes if ooc else 1) * a.numel() * 8 / dt / 1e9:.1f} GB/s H2D; sigma[:3] {s[:3].tolist()}", flush=True)
