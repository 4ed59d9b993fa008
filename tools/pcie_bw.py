"""Pinned host <-> device copy bandwidth (CUDA events), the bound of bench.py's e2e figure.

    python tools/pcie_bw.py [--gb 1.6]
"""
import argparse

import torch

p = argparse.ArgumentParser()
p.add_argument("--gb", type=float, default=1.6)
a = p.parse_args()
n = int(a.gb * 1e9 / 8)
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for name, dst, src in (("h2d", d, h), ("d2h", h, d)):
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{name} {a.gb:.2f} GB: {ms:.2f} ms = {a.gb / ms * 1e3:.1f} GB/s", flush=True)
