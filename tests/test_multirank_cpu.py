"""World-size-2 CPU (gloo) tests of the N>1 path's host-side logic.

The GPU path runs one process per GPU: every rank streams its own row shard,
the small partials (Gram matrix, column sums of squares, A^T Q) are
sum-allreduced, and every small core is recomputed redundantly on each rank.
These tests replay exactly that data flow with the oracle's step functions and
gloo allreduces, and check (a) it reproduces the single-process oracle and (b)
replicated results are bit-identical on every rank; plus bench.py's torchrun
launch (rank 0 prints one line, the other ranks exit 0).
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    sys.path.insert(0, ROOT)
    import oracle
    import synth
    from paper_1612_08709_b200 import shard_rows

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d = synth.config_inputs("c2", m=60_000)
        r0, r1 = shard_rows(60_000, world, rank)
        a = d["A"][r0:r1]
        wp = 1e-11

        def allreduce(x):
            t = torch.from_numpy(np.ascontiguousarray(x))
            dist.all_reduce(t)
            return t.numpy()

        # Alg. 4 with the GPU path's decomposition: local partial -> allreduce -> replicated core
        b = allreduce(a.T @ a)
        b = np.tril(b) + np.tril(b, -1).T  # symmetrise as the GPU path does after NCCL
        _, vt = oracle.sym_eig(b)
        yt = a @ vt
        st = np.sqrt(allreduce(np.sum(yt * yt, axis=0)))
        keep = oracle.keep_mask(st, wp)
        y = yt[:, keep] / st[keep]
        z = allreduce(y.T @ y)
        z = np.tril(z) + np.tril(z, -1).T
        _, w = oracle.sym_eig(z)
        qt = y @ w
        t = np.sqrt(allreduce(np.sum(qt * qt, axis=0)))
        keep2 = oracle.keep_mask(t, wp)
        q = qt[:, keep2] / t[keep2]
        rmat = (t[keep2][:, None] * w[:, keep2].T) @ (st[keep][:, None] * vt[:, keep].T)
        p, sig, vh = np.linalg.svd(rmat, full_matrices=False)
        u = q @ p
        # orthonormality of the distributed U, measured with an allreduced Gram
        g = allreduce(u.T @ u)
        out_q.put((rank, sig, vh, float(np.max(np.abs(g - np.eye(g.shape[0]))))))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_dataflow_matches_single_process_oracle():
    import oracle
    import synth

    world, port = 2, free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, s0, v0, o0), (_, s1, v1, o1) = res
    assert np.array_equal(s0, s1) and np.array_equal(v0, v1)  # replicated cores agree bitwise
    assert o0 <= 1e-13
    d = synth.config_inputs("c2", m=60_000)
    _, sr, _ = oracle.tssvd(d["A"], 1e-11, 2)
    assert s0.size == sr.size == 55
    assert np.max(np.abs(s0 - sr)) <= 1e-12


def test_bench_reference_arm_under_torchrun_two_ranks():
    """bench.py --impl reference launched like the driver does for N>1 (gloo on CPU)."""
    port = free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl",
           "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--cpu-sample-rows",
           "20000"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["n_gpus"] == 2 and rec["value"] > 0
    assert rec["cpu_baseline"]["kind"] == "oracle"
    assert rec["e2e"]["h2d_bytes_per_step"] == 0
