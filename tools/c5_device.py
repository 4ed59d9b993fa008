"""BASELINE configs[4] (c5: 500,000 x 40,000 FP64 = 160 GB, Alg. 8 with k = 50, l = 60, i = 4) on
ONE B200.  BASELINE lists c5 for 2/4/8 GPUs; one B200's 180 GB still holds A, so this runs it on
one device.  The 160 GB do not fit the host, so A is built on the device with torch's generator
following the same recipe as synth (A = U_r diag(sigma) V_r^T + 1e-8 G / sqrt(n), U_r and V_r Haar,
sigma_j = exp(-(j-1)/15), r = 100) -- same distribution, different bytes, so there is no oracle at
this size: the checks are properties (sigma_1..k against the constructed spectrum, U and V
orthonormal, the spectral error of the rank-k factors by 20 power iterations against
sigma_{k+1}).

    python tools/c5_device.py [--steps 3]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1612_08709_b200 as tk  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--m", type=int, default=500_000)
    p.add_argument("--n", type=int, default=40_000)
    a = p.parse_args()
    m, n, r, k, l, iters = a.m, a.n, 100, 50, 60, 4
    dev = torch.device("cuda", 0)
    f64 = torch.float64
    g = torch.Generator(device=dev).manual_seed(5)
    ur, _ = torch.linalg.qr(torch.randn(m, r, generator=g, device=dev, dtype=f64))
    vr, _ = torch.linalg.qr(torch.randn(n, r, generator=g, device=dev, dtype=f64))
    sigma = torch.exp(-torch.arange(r, device=dev, dtype=f64) / 15.0)
    b = sigma[:, None] * vr.T  # r x n
    A = torch.empty((m, n), device=dev, dtype=f64)
    step = 2048
    for i in range(0, m, step):
        j = min(m, i + step)
        torch.randn((j - i, n), generator=g, device=dev, dtype=f64, out=A[i:j])
        A[i:j].mul_(1e-8 / math.sqrt(n)).addmm_(ur[i:j], b)
    del ur, vr, b
    omega = torch.randn((n, l), generator=g, device=dev, dtype=f64)
    torch.cuda.synchronize()

    U, S, V = tk.lowrank_svd(A, omega, iters, k)  # warm-up
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.steps):
        U, S, V = tk.lowrank_svd(A, omega, iters, k)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps

    # properties
    sig = sigma[:k]
    dsig = (S - sig).abs().max().item()
    eye = torch.eye(k, device=dev, dtype=f64)
    ortho_u = (U.T @ U - eye).abs().max().item()
    ortho_v = (V.T @ V - eye).abs().max().item()
    x = torch.randn(n, generator=g, device=dev, dtype=f64)
    for _ in range(20):  # x <- M^T M x / |.|, M = A - U S V^T (never formed)
        y = A @ x - U @ (S * (V.T @ x))
        x = A.T @ y - V @ (S * (U.T @ y))
        x /= torch.linalg.norm(x)
    err = torch.linalg.norm(A @ x - U @ (S * (V.T @ x))).item()
    bytes_per_step = (2 * iters + 2) * A.numel() * 8
    print(json.dumps({
        "workload": f"c5 on one GPU: {m}x{n} FP64 ({A.numel() * 8 / 1e9:.0f} GB, built on the device), "
                    f"Alg. 8 k={k} l={l} i={iters}",
        "ms_per_step": round(ms, 2), "a_stream_GBps": round(bytes_per_step / ms / 1e6, 1),
        "max_abs_dsigma_1..k": dsig, "sigma_k+1": float(math.exp(-k / 15.0)),
        "spectral_error_20_power_iterations": err, "ortho_U": ortho_u, "ortho_V": ortho_v,
        "stats": tk.last_stats()}), flush=True)


if __name__ == "__main__":
    main()
