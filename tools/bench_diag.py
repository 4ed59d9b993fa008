"""Where does bench.py's c3 step time go?  Device-timed lowrank_svd steps (CUDA events on the
stream around K calls) with and without per-pass timing events and the nvidia-smi clock sampler.

    python tools/bench_diag.py [--steps 5]
"""
import argparse
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1612_08709_b200 as tk  # noqa: E402
from paper_1612_08709_b200 import _lib  # noqa: E402
import synth  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--config", default="c3")
    a = p.parse_args()
    cfg = synth.CONFIGS[a.config]
    d = synth.config_inputs(a.config)
    A = torch.from_numpy(d["A"]).cuda()
    Om = torch.from_numpy(d["Omega"]).cuda()
    s = torch.cuda.current_stream()

    def run(tag, timing, smi):
        _lib.set_pass_timing(timing)
        proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader",
                                 "-lms", "200"], stdout=subprocess.DEVNULL) if smi else None
        for _ in range(2):
            tk.lowrank_svd(A, Om, cfg["iters"], cfg["k"])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s)
        for _ in range(a.steps):
            tk.lowrank_svd(A, Om, cfg["iters"], cfg["k"])
        e1.record(s)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3 / a.steps
        if proc:
            proc.terminate()
            proc.wait()
        _lib.set_pass_timing(False)
        print(f"{tag:28s} device {e0.elapsed_time(e1) / a.steps:8.3f} ms/step  wall {wall:8.3f}", flush=True)

    for rep in range(2):
        run("plain", False, False)
        run("pass timing", True, False)
        run("nvidia-smi sampler", False, True)
        run("pass timing + sampler", True, True)


if __name__ == "__main__":
    main()
