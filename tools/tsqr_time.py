"""Device time of tsqr_svd (Alg. 1/2) and lowrank_svd_tsqr (Alg. 7) on BASELINE-shaped inputs,
with the per-pass CUDA-event split (tssvd_set_pass_timing)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1612_08709_b200 as tk
import synth
from paper_1612_08709_b200._lib import set_pass_timing

dev = torch.device("cuda", 0)


def timeit(f, reps=5):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), sorted(ts)[len(ts) // 2]


def passes_line():
    st = tk.last_stats()
    agg = {}
    for p in st["passes"]:
        agg.setdefault(p["kind"], [0, 0.0])
        agg[p["kind"]][0] += 1
        agg[p["kind"]][1] += p["ms"]
    return {k: (v[0], round(v[1], 3)) for k, v in agg.items()}


which = sys.argv[1:] or ["c2", "c3"]
for cfg in which:
    if cfg in ("c1", "c2", "c4"):
        c = synth.CONFIGS[cfg]
        m, n = c["m"], c["n"]
        if n > 128:
            continue
        A = torch.randn((m, n), dtype=torch.float64, device=dev)
        ph, pm = synth.mixing_params(n, 1)
        dph, dpm = torch.from_numpy(ph).to(dev), torch.from_numpy(pm).to(dev)
        for passes in (1, 2):
            t = timeit(lambda: tk.tsqr_svd(A, dph, dpm, passes=passes))
            set_pass_timing(True)
            tk.tsqr_svd(A, dph, dpm, passes=passes)
            torch.cuda.synchronize()
            set_pass_timing(False)
            pl = passes_line()
            tg = timeit(lambda: tk.tssvd(A, passes=passes))
            print(f"{cfg} m={m} n={n} alg{passes} tsqr min/med {t[0]:.2f}/{t[1]:.2f} ms; gram-based alg{passes + 2} "
                  f"{tg[0]:.2f}/{tg[1]:.2f} ms; tsqr passes {pl}", flush=True)
    else:
        c = synth.CONFIGS[cfg]
        m, n, l = c["m"], c["n"], c["l"]
        A = torch.randn((m, n), dtype=torch.float64, device=dev)
        Om = torch.randn((n, l), dtype=torch.float64, device=dev)
        ph, pm = tk.mixing_tables(lambda w: synth.mixing_params(w, 3), l, dev)
        t = timeit(lambda: tk.lowrank_svd_tsqr(A, Om, c["iters"], ph, pm, k=c["k"]))
        set_pass_timing(True)
        tk.lowrank_svd_tsqr(A, Om, c["iters"], ph, pm, k=c["k"])
        torch.cuda.synchronize()
        set_pass_timing(False)
        pl = passes_line()
        tg = timeit(lambda: tk.lowrank_svd(A, Om, c["iters"], k=c["k"]))
        tl = timeit(lambda: tk.lowrank_svd(A, Om, c["iters"], k=c["k"], tracking="lu"))
        set_pass_timing(True)
        tk.lowrank_svd(A, Om, c["iters"], k=c["k"], tracking="lu")
        torch.cuda.synchronize()
        set_pass_timing(False)
        pll = passes_line()
        print(f"{cfg} alg7 min/med {t[0]:.2f}/{t[1]:.2f} ms; alg8 {tg[0]:.2f}/{tg[1]:.2f} ms; passes {pl}",
              flush=True)
        print(f"{cfg} alg8 with LU tracking min/med {tl[0]:.2f}/{tl[1]:.2f} ms; passes {pll}", flush=True)
