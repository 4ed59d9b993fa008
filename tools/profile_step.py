"""Run a few tall-skinny SVD (or low-rank) steps for ncu captures.

    python tools/profile_step.py [--config c2] [--steps 2] [--m ROWS]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1612_08709_b200 as tk  # noqa: E402
import synth  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c2")
    p.add_argument("--steps", type=int, default=2)
    p.add_argument("--m", type=int, default=0)
    p.add_argument("--n", type=int, default=0)
    a = p.parse_args()
    cfg = synth.CONFIGS[a.config]
    d = synth.config_inputs(a.config, m=a.m or None, n=a.n or None)
    A = torch.from_numpy(d["A"]).cuda()
    for _ in range(a.steps):
        if cfg["kind"] == "tssvd":
            U = torch.empty_like(A)
            out = tk.tssvd(A, U=U)
        else:
            out = tk.lowrank_svd(A, torch.from_numpy(d["Omega"]).cuda(), cfg["iters"], cfg["k"])
    torch.cuda.synchronize()
    print("ok rank", out[1].numel(), tk.last_stats())


if __name__ == "__main__":
    main()
