"""Benchmark of the Gram-based SVD hot path on B200 (driver contract: one JSON line).

  python bench.py [--gpus N --steps K --warmup W] [--config c3] [--impl ours|reference]

A "step" is one whole call of the hot path on a BASELINE.json config, row-sharded
over N GPUs (strong scaling: the matrix is fixed).  Default: configs[2] (c3:
200,000 x 20,000 FP64, 32 GB, Alg. 8 randomized low-rank SVD, k=20 l=25 i=2) --
BASELINE's metric names no config, so the N=1 line runs the largest config that
BASELINE lists for 1 GPU; `--config c2` / `c4` run Alg. 4 on configs[1] / [3];
`--config c5` (configs[4], 160 GB, listed for 2/4/8 GPUs: A does not fit the host)
builds each rank's rows of A on its device (same recipe, torch's device generator).
`value` = A-stream throughput: algorithmic bytes of A streamed by the step's
passes over A (2 for Alg. 4: the Gram pass and the A V~ pass; 2i+2 for Alg. 8)
divided by the step time, summed over GPUs (whole job).
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def fp64_peak():
    """FP64 tensor (DMMA.8x8x4) peak measured on this pool's B200 by tools/fp64_peak.cu, committed
    as profiles/fp64_peak.json (MEASURED_PEAKS.json, driver-written, has no FP64 entry)."""
    d = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
    return d["dmma_tflops_sustained"], d


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="c3")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--wp", type=float, default=1e-11)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-clocks", action="store_true", help="diagnosis: no clock sampling")
    p.add_argument("--cpu-sample-rows", type=int, default=0)
    p.add_argument("--method", default="gram", choices=["gram", "tsqr", "lu"],
                   help="gram: Alg. 4 / Alg. 8 (the north star); tsqr: Alg. 2 / Alg. 7 (randomized "
                        "TSQR, n <= 128 for tall-skinny configs); lu: Alg. 8 with LU-based tracking "
                        "(low-rank configs)")
    return p.parse_args()


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class NvmlClocks:
    """In-process NVML sampling (a thread with one persistent NVML handle; BENCH_CLOCKS=nvml):
    the same clocks line as Clocks below without an nvidia-smi process polling the driver."""

    def __init__(self, index: int):
        self.index = index
        self.rows, self.th, self.stop_ev = [], None, None

    def start(self):
        import threading

        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            return
        bits = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
        self.stop_ev = threading.Event()

        def run():
            while not self.stop_ev.is_set():
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((time.time(), sm, mx, ["Active" if rs & b else "Not Active" for b in bits]))
                except Exception:
                    pass
                self.stop_ev.wait(0.2)

        self.th = threading.Thread(target=run, daemon=True)
        self.th.start()

    def mark_begin(self):
        self.t_begin = time.time()

    def mark_end(self):
        time.sleep(0.25)
        self.t_end = time.time()

    def stop(self):
        if not self.th:
            return None
        self.stop_ev.set()
        self.th.join()
        tb, te = getattr(self, "t_begin", 0.0), getattr(self, "t_end", time.time())
        rows = [r for r in self.rows if tb <= r[0] <= te] or self.rows
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, _, r in rows for i, v in enumerate(r) if v == "Active"})
        return {"sm_mhz": statistics.median(r[1] for r in rows), "sm_max_mhz": max(r[2] for r in rows),
                "reasons": reasons, "samples": len(rows), "sampler": "nvml"}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"bench_clocks_{os.getpid()}.csv")

    # The sampler is started BEFORE the warm-up steps: nvidia-smi's NVML start-up stalls the
    # GPU for tens of ms (measured r2: a c3 line of 54.5 ms/step when it started right at the
    # timed region, 46-47 ms/step with it running), so only its steady-state samples fall in
    # the timed window [mark_begin, mark_end], and only those are reported.
    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        self.t_begin = self.t_end = None

    def mark_begin(self):
        self.n_begin = self._count()

    def mark_end(self):
        time.sleep(0.25)
        self.n_end = self._count()

    def _count(self):
        try:
            return sum(1 for _ in open(self.path))
        except OSError:
            return 0

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        self.proc.wait()
        rows = []
        lines = open(self.path).read().splitlines()
        nb, ne = getattr(self, "n_begin", 0), getattr(self, "n_end", len(lines))
        window = lines[nb:ne] if ne > nb else lines[nb:] or lines
        for line in window:
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 7:
                try:
                    rows.append((float(f[0]), float(f[1]), f[3:7]))
                except ValueError:
                    pass
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v == "Active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


PASS_KERNEL = {"xv": "gemm_nn_kernel", "qnorm": "gemm_nn_kernel", "uout": "gemm_nn_kernel",
               "alpha": "gemm_nn_kernel", "gram_x": "syrk_kernel", "gram_y": "syrk_kernel",
               "beta": "gemm_tn_kernel"}


def ncu_traffic(config, kind):
    """(DRAM bytes per launch (read + write), source file) of a pass's kernel, from the committed
    ncu --set full capture of this workload (profiles/r0N_<config>_ncu_full_summary.txt, newest
    round first; first matching launch in step order), or (None, None) without a capture."""
    name = PASS_KERNEL.get(kind)
    paths = [os.path.join(ROOT, "profiles", f"r0{r}_{config}_ncu_full_summary.txt") for r in (2, 1)]
    path = next((p for p in paths if os.path.exists(p)), None)
    if not name or not path:
        return None, None
    order = ["gram_x", "xv", "gram_y", "qnorm", "uout"]  # launch order of one tssvd call
    want = [k for k in order if PASS_KERNEL.get(k) == name].index(kind) if kind in order else 0
    seen = 0
    for line in open(path):
        if line.startswith(name):
            if seen == want:
                try:
                    return round((_gbytes(line, "dram_rd=") + _gbytes(line, "dram_wr=")) * 1e9), \
                        os.path.relpath(path, ROOT)
                except (IndexError, ValueError):
                    return None, None
            seen += 1
    return None, None


def _gbytes(line, key):
    v = line.split(key)[1].split()[0]
    for unit, f in (("Gbyte", 1.0), ("Mbyte", 1e-3), ("Kbyte", 1e-6), ("byte", 1e-9)):
        if v.endswith(unit):
            return float(v[:-len(unit)]) * f
    return float(v)


def a_passes(cfg, method="gram"):
    # passes over A itself: Alg. 4 two Gram passes; Alg. 2 one (B* = A Omega*; its TSQRs work on
    # B* / Q); Alg. 5 + 6 (any factorization): 2 i + 2
    if cfg["kind"] == "tssvd":
        return 1 if method == "tsqr" else 2
    return 2 * cfg["iters"] + 2


MIX_SEED = 17  # the draws of Omega = D F S D~ F S~ for the TSQR-based algorithms


def oracle_step(oracle, cfg, d, a, method, wp):
    if cfg["kind"] == "tssvd":
        if method == "tsqr":
            oracle.tsqr_svd(a, *synth.mixing_params(a.shape[1], MIX_SEED), wp, 2)
        else:
            oracle.tssvd(a, wp, 2)
    elif method == "tsqr":
        oracle.lowrank_svd_tsqr(a, d["Omega"], d["iters"], d["k"], lambda w: synth.mixing_params(w, MIX_SEED), wp)
    elif method == "lu":
        oracle.lowrank_svd_lu(a, d["Omega"], d["iters"], d["k"], wp)
    else:
        oracle.lowrank_svd(a, d["Omega"], d["iters"], d["k"], wp)


# ------------------------------------------------------------ reference --
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args, rank, world):
    """--impl reference: the oracle (oracle/) as it stands, on the host cores, bounded samples."""
    if rank != 0:
        return
    import oracle

    cfg = synth.CONFIGS[args.config]
    rows = args.cpu_sample_rows or (min(200_000, max(10_000, int(2e11 / cfg["n"] ** 2)))
                                     if cfg["kind"] == "tssvd" else 20_000)
    d = synth.config_inputs(args.config, m=min(rows, cfg["m"]),
                            n=None if cfg["kind"] == "tssvd" else min(cfg["n"], 4_000))
    a = d["A"]

    def step():
        oracle_step(oracle, cfg, d, a, args.method, cfg.get("wp", args.wp))

    for _ in range(args.warmup):
        step()
    t0, c0 = time.perf_counter(), time.process_time()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    cpu_s = (time.process_time() - c0) / args.steps
    gbs = a_passes(cfg, args.method) * a.nbytes / dt / 1e9
    sample = f"first {a.shape[0]} rows x {a.shape[1]} cols of {args.config} ({a.nbytes / 1e9:.2f} GB)"
    line = {"impl": "reference", "metric": metric_name(cfg, args.method), "value": round(gbs, 3), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_obj(args, cfg, world),
            "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": os.cpu_count(),
                             "kind": "oracle", "sample": sample, "cpu_model": cpu_model(),
                             "wall_s_per_step": round(dt, 3), "cpu_s_per_step": round(cpu_s, 3)},
            "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def metric_name(cfg, method="gram"):
    if cfg["kind"] == "tssvd":
        return "A-stream GB/s (Alg. 2 TSQR-based tall-skinny SVD)" if method == "tsqr" else \
            "A-stream GB/s (Alg. 4 tall-skinny SVD)"
    return {"tsqr": "A-stream GB/s (Alg. 7 low-rank SVD)",
            "lu": "A-stream GB/s (Alg. 8 low-rank SVD, LU-based tracking)"}.get(
        method, "A-stream GB/s (Alg. 8 low-rank SVD)")


def config_obj(args, cfg, world):
    paper = {"t3": "PAPER Table 3", "t4": "PAPER Table 4", "t5": "PAPER Table 5",
             "s21": "PAPER Table 21 (Devil's staircase)"}.get(args.config)
    alg_t = "Alg. 2 (random mixing, two TSQRs)" if args.method == "tsqr" else "Alg. 4 (two Gram passes)"
    alg_l = {"tsqr": "Alg. 7", "lu": "Alg. 8 with LU-based tracking (P:405-409)"}.get(args.method, "Alg. 8")
    c = {"workload": f"{args.config}: {cfg['m']}x{cfg['n']} FP64 "
                     + (f"tall-skinny SVD, {alg_t}" if cfg["kind"] == "tssvd"
                        else f"low-rank SVD {alg_l}, k={cfg['k']} l={cfg['l']} i={cfg['iters']}")
                     + (f", {paper} matrix (Eq. originalmat, DCT factors)" if paper else ""),
         "m": cfg["m"], "n": cfg["n"], "rows_per_gpu": -(-cfg["m"] // world),
         "working_precision": cfg.get("wp", args.wp), "parallelism": f"row-shard x{world}",
         "l2": "A is larger than L2 (126 MB) on every rank; no flush needed"}
    if args.config in DEVICE_BUILT and args.impl == "ours":
        c["inputs"] = ("A and Omega built on each rank's device by torch's generator (the synth "
                       "recipe's distribution, not its bytes; A does not fit the host)")
    return c


# ------------------------------------------------------------ ours -------
DEVICE_BUILT = ("c5",)  # A too large for the host: built on the device (inputs only, no method)


def device_lowrank_inputs(cfg, r0, r1, world, rank, dev):
    """Rows [r0, r1) of A = U_r diag(sigma) V_r^T + noise G / sqrt(n) and Omega, built on `dev`
    with torch's device generator (the synth recipe's distribution, other bytes: there is no
    oracle at this size).  V_r, sigma and Omega are identical on every rank (common seed); the
    rank's block of U_r is Q_p / sqrt(P) with Q_p the QR factor of the rank's own Gaussian block,
    so U_r^T U_r = sum_p Q_p^T Q_p / P = I (orthonormal; Haar for P = 1)."""
    import math

    import torch

    f64 = torch.float64
    m_local, n, r = r1 - r0, cfg["n"], cfg["r"]
    gc_ = torch.Generator(device=dev).manual_seed(cfg["seed"])
    vr, _ = torch.linalg.qr(torch.randn(n, r, generator=gc_, device=dev, dtype=f64))
    omega = torch.randn((n, cfg["l"]), generator=gc_, device=dev, dtype=f64)
    sigma = torch.from_numpy(synth.spectrum(cfg["spec"][0], r)).to(dev)
    b = sigma[:, None] * vr.T  # r x n
    del vr
    gr = torch.Generator(device=dev).manual_seed(cfg["seed"] * 1000 + 1 + rank)
    ur, _ = torch.linalg.qr(torch.randn(m_local, r, generator=gr, device=dev, dtype=f64))
    ur /= math.sqrt(world)
    A = torch.empty((m_local, n), device=dev, dtype=f64)
    step = 2048
    for i in range(0, m_local, step):
        j = min(m_local, i + step)
        torch.randn((j - i, n), generator=gr, device=dev, dtype=f64, out=A[i:j])
        A[i:j].mul_(cfg["noise"] / math.sqrt(n)).addmm_(ur[i:j], b)
    del ur, b
    if dev.type == "cuda":
        torch.cuda.synchronize(dev)
    return A, omega


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1612_08709_b200 as tk
    from paper_1612_08709_b200 import _lib

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    comm = tk.Comm(device=local_rank) if world > 1 else None
    cfg = synth.CONFIGS[args.config]
    r0, r1 = tk.shard_rows(cfg["m"], world, rank)
    lowrank = cfg["kind"] == "lowrank"
    device_built = args.config in DEVICE_BUILT
    if device_built:
        if args.method != "gram":
            raise SystemExit(f"--config {args.config}: device-built inputs run the Gram-based method only")
        A, Om = device_lowrank_inputs(cfg, r0, r1, world, rank, dev)
        a_host = om_host = None
    else:
        d = synth.config_inputs(args.config, rows=(r0, r1))
        # the pinned copy is the only host A kept (the e2e leg's input): the generator's array is
        # released before any timing (c3: 32 GB), and the host gets a moment to settle after the
        # large allocations -- first c3 runs on a fresh box showed 10 ms/step of host-side GPU idle
        a_host = torch.from_numpy(d.pop("A")).pin_memory()
        A = a_host.to(dev)
        if lowrank:
            om_host = torch.from_numpy(d["Omega"]).pin_memory()
            Om = om_host.to(dev)
    gc.collect()
    torch.cuda.synchronize()
    time.sleep(1.0)
    m_local, n = A.shape
    U = torch.empty_like(A) if not lowrank else None

    wp = cfg.get("wp", args.wp)  # the paper workloads fix their own (reading Q1)
    method = args.method
    if method == "tsqr" and not lowrank and n > 128:
        raise SystemExit(f"--method tsqr: tall-skinny configs need n <= 128 ({args.config} has n = {n})")
    if method == "lu" and not lowrank:
        raise SystemExit("--method lu applies to the low-rank configs")
    if method == "tsqr":
        if lowrank:
            ph, pm = tk.mixing_tables(lambda w: synth.mixing_params(w, MIX_SEED), cfg["l"], dev)
        else:
            ph_np, pm_np = synth.mixing_params(n, MIX_SEED)
            ph, pm = torch.from_numpy(ph_np).to(dev), torch.from_numpy(pm_np).to(dev)

    def step():
        if lowrank:
            if method == "tsqr":
                return tk.lowrank_svd_tsqr(A, Om, cfg["iters"], ph, pm, k=cfg["k"], wp=wp, comm=comm)
            return tk.lowrank_svd(A, Om, cfg["iters"], cfg["k"], wp=wp, comm=comm,
                                  tracking="lu" if method == "lu" else "q")
        if method == "tsqr":
            return tk.tsqr_svd(A, ph, pm, wp=wp, passes=2, comm=comm)
        return tk.tssvd(A, wp=wp, passes=2, comm=comm, U=U)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = NvmlClocks(local_rank) if os.environ.get("BENCH_CLOCKS") == "nvml" else Clocks(local_rank)
    if not args.no_clocks:
        clocks.start()
    # pass timing on already in the warm-up: it is part of a call's CUDA-graph key, and the
    # warm-up must capture the graphs the timed steps replay (the outputs of consecutive calls
    # alternate between two buffer sets: >= 2 warm-up steps capture both).  Switching it on at
    # the timed region made the first timed steps capture + instantiate their graphs inside the
    # timed region (c3: up to 10 ms/step of GPU idle in some runs).
    _lib.set_pass_timing(True)
    for _ in range(args.warmup):
        out = step()
    st = _lib.last_stats()
    launches = st["kernel_launches"]
    barrier()
    clocks.mark_begin()
    pass_ms = {}
    pass_flops = {}
    pass_kinds, pass_bytes = [], []
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    raws = []
    for _ in range(args.steps):
        out = step()
        raws.append(_lib.raw_stats())  # decoded after the timed region (host time between calls)
    e1.record(stream)
    barrier()
    for raw in raws:
        for p in _lib.decode_stats(raw)["passes"]:
            pass_ms.setdefault(p["kind"], []).append(p["ms"])
            pass_flops.setdefault(p["kind"], []).append(p["flops"])
            pass_kinds.append(p["kind"])
            pass_bytes.append(p["bytes"])
    clocks.mark_end()
    _lib.set_pass_timing(False)
    ck = clocks.stop()
    t = e0.elapsed_time(e1) / args.steps  # ms per step on this rank
    tt = torch.tensor([t], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t = tt.item()
    total_a_bytes = 8.0 * cfg["m"] * cfg["n"] * a_passes(cfg, method)
    value = total_a_bytes / (t * 1e-3) / 1e9

    # e2e through the same C-ABI call with HOST buffers (H2D of A, D2H of U/sigma/V inside)
    e2e = None
    if method == "tsqr":
        e2e = {"value": None, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
               "unavailable": "the TSQR entry points take device pointers only (host_io 0)"}
    elif device_built:
        e2e = {"value": None, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
               "unavailable": f"{args.config}'s A ({8 * cfg['m'] * cfg['n'] / 1e9:.0f} GB) does not fit "
                              "the host: built on the device, no host copy to stream"}
    elif not args.no_e2e:
        ts = []
        ew = max(2, min(args.warmup, 3))  # >= 2: the pinned output blocks of two calls are live
        for i in range(ew + args.steps):
            barrier()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            if lowrank:
                u_h, s_h, v_h = tk.lowrank_svd(a_host, om_host, cfg["iters"], cfg["k"], wp=wp,
                                               comm=comm, tracking="lu" if method == "lu" else "q")
            else:
                u_h, s_h, v_h = tk.tssvd(a_host, wp=wp, passes=2, comm=comm)
            s1.record(stream)
            s1.synchronize()
            if i >= ew:
                ts.append(s0.elapsed_time(s1))
        te = torch.tensor([statistics.mean(ts)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        r = u_h.shape[1]
        h2d = 8 * m_local * n + (8 * om_host.numel() if lowrank else 0)
        d2h = 8 * (m_local * r + r + n * r) if lowrank else 8 * (m_local * ((r + 1) & ~1) + r + n * r)
        e2e = {"value": round(total_a_bytes / (te.item() * 1e-3) / 1e9, 3), "unit": "GB/s",
               "ms_per_step": round(te.item(), 3), "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h),
               "path": "the same C-ABI call with pinned HOST buffers (opts.host_io = 1): H2D of A"
                       + (" and Omega" if lowrank else "") + ", compute, D2H of U, sigma, V -- "
                       "all inside the timed region (PCIe-bound)"}

    # roofline of the dominant kernel (largest share of the step's device time), plus every
    # streaming pass's own fraction; the Jacobi cores (latency-bound, no roofline) by share
    peak, peak_info = fp64_peak()
    shares = {k: sum(v) / args.steps for k, v in pass_ms.items()}
    dom = max((k for k in shares if k != "jacobi"), key=lambda k: shares[k])

    def rate(kind):
        return statistics.mean(pass_flops[kind]) / (statistics.mean(pass_ms[kind]) * 1e-3) / 1e12

    achieved = rate(dom)
    traffic, traffic_src = ncu_traffic(args.config, dom)
    roof = {"kernel": dom, "bound": "alu" if dom == "tsqr" else "tensor", "achieved": round(achieved, 3),
            "peak": peak, "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
            "traffic": traffic, "traffic_source": traffic_src,
            "algorithmic_bytes_per_launch": round(statistics.mean(
                [b for k, b in zip(pass_kinds, pass_bytes) if k == dom])) if pass_bytes else None,
            "peak_source": "FP64 DMMA.8x8x4 sustained throughput measured on this pool's B200 by "
                           "tools/fp64_peak.cu (profiles/fp64_peak.json; MEASURED_PEAKS.json has no "
                           "FP64 entry)",
            "share_of_step": round(shares[dom] / t, 4),
            "pass_ms_per_step": {k: round(v, 4) for k, v in sorted(shares.items())},
            "pass_frac": {k: round(rate(k) / peak, 4) for k in sorted(shares) if k != "jacobi"},
            "jacobi_share_of_step": round(shares.get("jacobi", 0.0) / t, 4)}

    # Alg. 3 vs Alg. 4 orthonormality (BASELINE configs[1]): max|U^T U - I| after one and after
    # two Gram passes, measured with a cuBLAS Gram outside the timed region
    ortho = None
    if not lowrank and world == 1 and method == "gram":
        ortho = {}
        for npass in (1, 2):
            u1, s1_, _ = tk.tssvd(A, wp=wp, passes=npass, U=U)
            g = u1.T @ u1
            ortho[f"pass{npass}"] = (g - torch.eye(g.shape[0], dtype=g.dtype, device=dev)).abs().max().item()

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, cfg)

    # context only (frac stays against the nominal-clock peak): the FP64 pipe's rate scales with the
    # SM clock, so under sw_power_cap the attainable peak is peak * sm_mhz / sm_max_mhz
    if ck and ck.get("sm_mhz") and ck.get("sm_max_mhz") and roof["bound"] == "tensor":
        roof["frac_at_sampled_clock"] = round(achieved / (peak * ck["sm_mhz"] / ck["sm_max_mhz"]), 4)

    if rank == 0:
        line = {"metric": metric_name(cfg, method), "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t, 4),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": config_obj(args, cfg, world),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": ck,
                "gpu_launches": int(launches * args.steps),
                "kept_rank": int(out[1].numel()),
                "ranks": st["ranks"],
                "jacobi_sweeps": st["jacobi_sweeps"]}
        if ortho is not None:
            line["ortho_UtU_minus_I"] = ortho
        print(json.dumps(line), flush=True)
    if comm:
        comm.close()


def cpu_baseline(args, cfg):
    """The oracle as it stands, on this host's cores, on a bounded sample (~10-30 s)."""
    import oracle

    # bounded sample: ~2e11 m n^2 for the tall-skinny configs (500,000 rows at n = 100,
    # 50,000 at n = 2000), 20,000 x 4,000 for the low-rank ones
    tall_rows = min(500_000, max(10_000, int(2e11 / cfg["n"] ** 2)))
    rows = args.cpu_sample_rows or (tall_rows if cfg["kind"] == "tssvd" else 20_000)
    d = synth.config_inputs(args.config, m=min(rows, cfg["m"]),
                            n=None if cfg["kind"] == "tssvd" else min(cfg["n"], 4_000))
    a = d["A"]
    reps, t0, c0 = 0, time.perf_counter(), time.process_time()
    while True:
        oracle_step(oracle, cfg, d, a, args.method, cfg.get("wp", args.wp))
        reps += 1
        if time.perf_counter() - t0 > 10.0 or reps >= 20:
            break
    dt = (time.perf_counter() - t0) / reps
    cpu_s = (time.process_time() - c0) / reps
    return {"value": round(a_passes(cfg, args.method) * a.nbytes / dt / 1e9, 3), "unit": "GB/s",
            "cores": os.cpu_count(), "kind": "oracle", "cpu_model": cpu_model(),
            "wall_s_per_step": round(dt, 3), "cpu_s_per_step": round(cpu_s, 3),
            "sample": f"{reps} oracle runs on the first {a.shape[0]} rows x {a.shape[1]} cols of "
                      f"{args.config} ({a.nbytes / 1e9:.2f} GB), {dt:.2f} s each"}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank) if args.impl == "ours" else None
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
