"""Per-step timing of lowrank_svd on c3 (device clock vs host wall) to find host gaps."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
if os.environ.get("LIBALT"):
    from paper_1612_08709_b200 import _lib as _l0
    _l0.LIB_PATH = os.environ["LIBALT"]
import paper_1612_08709_b200 as tk
from paper_1612_08709_b200 import _lib
import synth
m = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
d = synth.config_inputs("c3", m=m)
A = torch.from_numpy(d["A"]).cuda(); Om = torch.from_numpy(d["Omega"]).cuda()
_lib.set_pass_timing(True)
for it in range(int(os.environ.get("STEPS", "6"))):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    tk.lowrank_svd(A, Om, d["iters"], d["k"])
    e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
    st = _lib.last_stats()
    ps = sum(p["ms"] for p in st["passes"])
    kinds = {}
    for p in st["passes"]:
        kinds[p["kind"]] = kinds.get(p["kind"], 0.0) + p["ms"]
    print(f"step {it}: device {e0.elapsed_time(e1):.2f} ms, host {1e3 * (t1 - t0):.2f} ms, passes {ps:.2f} ms, launches {st['kernel_launches']} " + str({k: round(v, 2) for k, v in kinds.items()}), flush=True)
