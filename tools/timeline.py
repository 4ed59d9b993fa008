"""Device timeline of one call (CUPTI through torch.profiler): every kernel / memcpy of the
library on the stream, its duration, and the idle gaps between consecutive GPU activities.

    python tools/timeline.py [--config c3] [--steps 2] [--top 25]

Prints the step's device busy time vs. its wall span and the largest gaps with the activity
that follows each gap (what the GPU was waiting for).
"""
import argparse
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1612_08709_b200 as tk  # noqa: E402
import synth  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c3")
    p.add_argument("--steps", type=int, default=2)
    p.add_argument("--top", type=int, default=25)
    p.add_argument("--m", type=int, default=0)
    a = p.parse_args()
    cfg = synth.CONFIGS[a.config]
    d = synth.config_inputs(a.config, m=a.m or None)
    A = torch.from_numpy(d["A"]).cuda()
    lowrank = cfg["kind"] == "lowrank"
    Om = torch.from_numpy(d["Omega"]).cuda() if lowrank else None
    U = None if lowrank else torch.empty_like(A)

    def step():
        if lowrank:
            return tk.lowrank_svd(A, Om, cfg["iters"], cfg["k"])
        return tk.tssvd(A, U=U)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(a.steps):
            step()
        torch.cuda.synchronize()
    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    gpu.sort(key=lambda e: e["ts"])
    if not gpu:
        print("no GPU activity captured")
        return
    t0, t1 = gpu[0]["ts"], gpu[-1]["ts"] + gpu[-1]["dur"]
    busy = sum(e["dur"] for e in gpu)
    gaps = []
    for x, y in zip(gpu, gpu[1:]):
        g = y["ts"] - (x["ts"] + x["dur"])
        gaps.append((g, x["name"][:60], y["name"][:60]))
    gaps.sort(reverse=True)
    by = {}
    for e in gpu:
        k = e["name"].split("(")[0].split("<")[0].replace("void ", "")[:50]
        c, s = by.get(k, (0, 0.0))
        by[k] = (c + 1, s + e["dur"])
    print(json.dumps({"config": a.config, "steps": a.steps, "span_ms_per_step": (t1 - t0) / 1e3 / a.steps,
                      "busy_ms_per_step": busy / 1e3 / a.steps,
                      "idle_ms_per_step": (t1 - t0 - busy) / 1e3 / a.steps,
                      "activities_per_step": len(gpu) / a.steps}))
    print("by kernel (count, ms per step):")
    for k, (c, s) in sorted(by.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:52s} {c / a.steps:7.1f} {s / 1e3 / a.steps:9.4f}")
    print(f"largest gaps (us): before -> after")
    for g, x, y in gaps[: a.top]:
        print(f"  {g:9.1f}  {x} -> {y}")
    tot = sum(g for g, _, _ in gaps)
    small = sum(g for g, _, _ in gaps if g < 20)
    print(f"gaps total {tot / 1e3 / a.steps:.3f} ms/step, of which < 20 us each: {small / 1e3 / a.steps:.3f} ms/step")


if __name__ == "__main__":
    main()
