"""Time the Gram kernel alone at a given (m, w) with CUDA events.
    python tools/gram_bench.py --m 2000000 --w 200 [--lib path.so]"""
import argparse, os, sys, ctypes
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
p = argparse.ArgumentParser()
p.add_argument("--m", type=int, default=2_000_000)
p.add_argument("--w", type=int, nargs="*", default=[200])
p.add_argument("--lib", default="")
a = p.parse_args()
if a.lib:
    from paper_1612_08709_b200 import _lib
    _lib.LIB_PATH = a.lib
import paper_1612_08709_b200 as tk
for w in a.w:
    X = torch.randn(a.m, w + (w & 1), dtype=torch.float64, device="cuda")[:, :w]
    tk.gram(X)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        tk.gram(X)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"w={w} m={a.m} gram ms={ms:.3f} TF={a.m * w * (w + 1) / ms / 1e9:.1f}", flush=True)
