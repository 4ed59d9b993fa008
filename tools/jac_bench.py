"""Time the small-core Jacobi kernels alone (CUDA events), for ncu captures too.

    python tools/jac_bench.py [--n 100 55] [--reps 5]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1612_08709_b200 as tk  # noqa: E402


def graded_gram(n, decades, seed):
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = 10.0 ** (-decades * np.arange(n) / max(n - 1, 1))
    return (q * s**2) @ q.T


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--n", type=int, nargs="*", default=[100, 55, 200])
    p.add_argument("--reps", type=int, default=5)
    a = p.parse_args()
    for n in a.n:
        b = torch.from_numpy(graded_gram(n, 10, n)).cuda()
        lam, v, sw = tk.sym_eig(b)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.reps):
            tk.sym_eig(b)
        e1.record()
        torch.cuda.synchronize()
        ws = tk.api._ws_cache[("cuda", 0)]
        info = ws[n * n * 8:n * n * 8 + 40].view(torch.int32).cpu().tolist()
        chol_us, sw_us = info[3] * 16 / 1965.0, info[4] * 16 / 1965.0
        print(f"n={n} sweeps={sw} k={int((lam > 0).sum())} ms={e0.elapsed_time(e1) / a.reps:.3f} "
              f"chol_us={chol_us:.1f} sweeps_us={sw_us:.1f} rounds={info[5]} "
              f"cyc/round={info[4] * 16 / max(info[5], 1):.0f} G={os.environ.get('TSSVD_JAC_G', 'auto')}", flush=True)


if __name__ == "__main__":
    main()
