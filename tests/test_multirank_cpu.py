"""World-size-2 CPU (gloo) tests of the N>1 path's host-side logic.

The GPU path runs one process per GPU: every rank streams its own row shard,
the small partials (packed Gram matrix, column sums of squares, A^T Q) are
sum-allreduced, and every small core is recomputed redundantly on each rank.

These tests do not re-type that data flow: each rank asks the LIBRARY for the
exact step sequence its orchestrator (csrc/api.cu) would run on that rank
(`tssvd_trace`, a plan-only run that makes no CUDA or NCCL call), and replays
it token by token -- numpy for the local arithmetic (LAPACK standing in for the
Jacobi kernels), gloo allreduces for the collectives, with the message sizes
the trace announces.  Checks: (a) the replay reproduces the single-process
oracle, (b) replicated results are bit-identical on every rank, (c) every
collective's size is the one the replay needs (packed Gram w(w+1)/2, norms,
A^T Q without pad columns), (d) the host round trips are where the design says
(none before the end for lowrank_svd and narrow tssvd; two for wide tssvd);
plus bench.py's torchrun launch (rank 0 prints one line, the other ranks exit 0).
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
from parity import assert_lowrank_parity, assert_tssvd_parity

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WP = 1e-11


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class Replay:
    """Interprets the orchestrator's trace on one rank (numpy + gloo)."""

    def __init__(self, a_local, omega=None, mixes=None):
        import oracle

        self.o = oracle
        self.mixes = mixes      # width -> (phases, perms): the draws of Alg. 1/2's Omega
        self.a = a_local
        self.omega = omega
        self.collectives = []   # (what, count) as announced by the trace
        self.pending = None     # local partial awaiting its allreduce
        self.cur = None         # the core's input matrix
        self.dist = False
        self.out = {}           # outputs of the last finished core

    # -- LU-based tracking: distributed partial pivoting, one column per token
    def lu_local(self, j):
        lu = self.lu
        w = lu["W"]
        lu["j"] = j
        if lu["stopped"] or j >= w.shape[1]:
            lu["val"], lu["idx"] = -1.0, -1
            return
        mag = np.abs(w[:, j]) if w.shape[0] else np.zeros(0)
        if w.shape[0]:
            mag[lu["chosen"]] = -1.0
        lu["idx"] = int(np.argmax(mag)) if mag.size else -1
        lu["val"] = float(mag[lu["idx"]]) if mag.size else -1.0

    def lu_step(self, gmax, owner, urow):
        lu = self.lu
        j = lu["j"]
        w = lu["W"]
        if lu["stopped"] or j >= w.shape[1]:
            lu["stopped"] = True
            return
        if j == 0:
            lu["p1"] = max(gmax, 0.0)
        if not (lu["p1"] > 0.0 and gmax > lu["p1"] * WP):
            lu["stopped"] = True
            return
        mine = owner == (dist.get_rank() if self.dist else 0)
        pv = urow[-1]
        mult = w[:, j] / pv
        mult[lu["chosen"]] = 0.0
        if mine:
            mult[lu["idx"]] = 1.0
            lu["chosen"][lu["idx"]] = True
        lu["L"][:, j] = mult
        w[:, j + 1:] -= np.outer(mult, urow[j + 1:w.shape[1]])
        lu["r"] = j + 1

    def lu_allreduce(self, what, count):
        lu = self.lu
        if what == "lu_max":
            t = torch.tensor([lu["val"]], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            lu["gmax"] = float(t.item())
        elif what == "lu_owner":
            mine = lu["val"] >= 0.0 and lu["val"] == lu["gmax"]
            t = torch.tensor([dist.get_rank() if mine else 2 ** 31 - 1], dtype=torch.int32)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            lu["owner"] = int(t.item())
        else:  # lu_row: the owner's pivot row (+ the signed pivot), zeros elsewhere
            w = lu["W"]
            assert count >= w.shape[1] + 1, (count, w.shape)
            row = np.zeros(count)
            if lu["owner"] == dist.get_rank() and lu["idx"] >= 0 and lu["j"] < w.shape[1]:
                row[:w.shape[1]] = w[lu["idx"]]
                row[count - 1] = w[lu["idx"], lu["j"]]
            t = torch.from_numpy(row)
            dist.all_reduce(t)
            u = t.numpy()
            self.lu_step(lu["gmax"], lu["owner"], np.concatenate([u[:w.shape[1]], u[count - 1:]]))

    # -- collectives
    def allreduce(self, what, count):
        if what.startswith("lu_"):
            self.collectives.append((what, count))
            return self.lu_allreduce(what, count)
        self.collectives.append((what, count))
        if what == "m":
            t = torch.tensor([self.a.shape[0]], dtype=torch.int64)
            dist.all_reduce(t)
            self.m = int(t.item())
            return
        # a plan-only trace carries the launch BOUNDS (a dry run's decisions keep every
        # column), so a message is at least as large as the data the replay reduces
        x = self.pending
        if what == "gram":  # packed lower triangle on the wire
            w = x.shape[0]
            assert count >= w * (w + 1) // 2, (what, count, w)
            il = np.tril_indices(w)
            t = torch.from_numpy(np.ascontiguousarray(x[il]))
            dist.all_reduce(t)
            full = np.zeros_like(x)
            full[il] = t.numpy()
            self.pending = np.tril(full) + np.tril(full, -1).T
        elif what == "norms":
            assert count >= x.size, (what, count, x.size)
            t = torch.from_numpy(np.ascontiguousarray(x))
            dist.all_reduce(t)
            self.pending = t.numpy()
        elif what == "beta":  # n x even(l): no partial pad columns
            n, l = x.shape
            assert count >= n * (l + (l & 1)) and count % n == 0 and (count // n) % 2 == 0, (count, x.shape)
            t = torch.from_numpy(np.ascontiguousarray(x))
            dist.all_reduce(t)
            self.pending = self.cur = t.numpy()
        else:
            raise AssertionError(f"unknown collective {what}")

    # -- Alg. 1 / 2 tokens (TSQR cores)
    def run_tsqr(self, tok):
        o = self.o
        parts = tok.split(":")
        k = parts[0]
        c = getattr(self, "c", {})
        if k == "tsqr_core":
            self.mode = "tsqr"
            self.dist = parts[1] == "sharded"
            self.passes = int(parts[2])
            self.x = self.cur if self.cur is not None else self.a
            self.c = {"R": []}
        elif k == "mix":  # B^* = every row mixed (the draws for this factorization's width)
            ph, pm = self.mixes(self.x.shape[1])
            c["ph"], c["pm"] = ph, pm
            c["q"] = o.mix_rows(self.x, ph, pm)
        elif k == "tsqr":  # the rank's local QR (the top of the tree follows if sharded)
            q, r = np.linalg.qr(c["q"], mode="reduced")
            c["q"], c["r"] = q, r
            if not self.dist:
                c["R"].append(r)
        elif k == "allgather":  # R_p of every rank, stacked in rank order, factored again
            w = c["r"].shape[1]
            count = int(parts[2])
            assert count >= w * w, (count, w)
            self.collectives.append(("allgather", count))
            rl = np.zeros((w, w))
            rl[:c["r"].shape[0]] = c["r"]
            bufs = [torch.zeros((w, w), dtype=torch.float64) for _ in range(dist.get_world_size())]
            dist.all_gather(bufs, torch.from_numpy(rl))
            stack = np.vstack([b.numpy() for b in bufs])
            qt, r = np.linalg.qr(stack, mode="reduced")
            rank = dist.get_rank()
            qloc = np.zeros((c["q"].shape[0], w))
            qloc[:, :c["q"].shape[1]] = c["q"]
            c["q"] = qloc @ qt[rank * w:(rank + 1) * w]
            c["R"].append(r)
        elif k == "discard":  # |R_jj| < |R_11| wp (reading R18); rows of R, columns of Q
            r = c["R"][-1]
            keep = o.r_keep(r, WP)
            c["q"], c["R"][-1] = c["q"][:, keep], r[keep, :]
        elif k == "zero_cols":  # Alg. 2: the kept Q~ is QR'd again
            pass
        elif k == "svd":
            mat = c["R"][0] if self.passes == 1 else c["R"][1] @ c["R"][0]
            ut, sig, vth = np.linalg.svd(mat, full_matrices=False)
            c["ut"], c["sig"], c["vth"] = ut, sig, vth
        elif k == "tsqr_out":
            c["U"], c["S"] = c["q"] @ c["ut"], c["sig"]
            c["V"] = o.mix_rows(c["vth"], c["ph"], c["pm"], inverse=True).T
        else:
            raise AssertionError(f"unknown tsqr token {tok}")

    # -- one token
    def run(self, tok):
        o = self.o
        parts = tok.split(":")
        k = parts[0]
        if k in ("tssvd", "lowrank", "finish", "sync", "build_z", "h2d", "d2h", "tsqr_svd", "tsqr_top"):
            return
        if k == "tsqr_core" or getattr(self, "mode", "") == "tsqr" and k in (
                "mix", "tsqr", "allgather", "discard", "zero_cols", "svd", "tsqr_out"):
            return self.run_tsqr(tok)
        if k == "allreduce":
            self.allreduce(parts[1], int(parts[2]))
        elif k == "lu_core":
            self.mode = "lu"
            self.dist = parts[1] == "sharded"
            x = self.cur if self.cur is not None else self.a
            self.lu = dict(W=np.array(x, dtype=np.float64), chosen=np.zeros(x.shape[0], dtype=bool),
                           L=np.zeros(x.shape), r=0, stopped=False, p1=0.0)
        elif k == "lu_col":
            self.lu_local(int(parts[1]))
            if not self.dist:  # single rank: the decision and the update right away
                lu = self.lu
                w = lu["W"]
                if lu["idx"] >= 0 and lu["j"] < w.shape[1]:
                    urow = np.concatenate([w[lu["idx"]], [w[lu["idx"], lu["j"]]]])
                else:
                    urow = np.zeros(w.shape[1] + 1)
                self.lu_step(lu["val"], 0, urow)
        elif k == "lu_finish":
            self.out = dict(U=self.lu["L"][:, :self.lu["r"]])
        elif k == "core":
            self.mode = "gram"
            self.dist = parts[1] == "sharded"
            self.passes = int(parts[2])
            self.x = self.cur if self.cur is not None else self.a
            self.c = {}
        elif k == "gram":
            src = self.x if parts[1] == "X" else self.c["y"]
            self.pending = src.T @ src
            self._settle = "B" if parts[1] == "X" else "Z"
        elif k == "eig":
            mat = self.pending
            _, v = o.sym_eig(mat)
            self.c["V~" if parts[1] == "B" else "W"] = v
        elif k == "xv":
            yt = self.x @ self.c["V~"]
            self.c["yt"] = yt
            self.pending = np.sum(yt * yt, axis=0)
        elif k == "discard":
            s = np.sqrt(self.pending)
            keep = o.keep_mask(s, WP)
            if parts[1] == "1":
                self.c.update(sig=s[keep], keep=keep)
                self.c["y"] = self.c["yt"][:, keep] / s[keep]
            else:
                self.c.update(t=s[keep], keep2=keep)
        elif k == "alg3_out":
            c = self.c
            order = np.argsort(-c["sig"], kind="stable")
            c["U"] = c["y"][:, order]
            c["S"] = c["sig"][order]
            c["V"] = c["V~"][:, c["keep"]][:, order]
        elif k == "qnorm":
            qt = self.c["y"] @ self.c["W"]
            self.c["qt"] = qt
            self.pending = np.sum(qt * qt, axis=0)
        elif k == "svd":
            c = self.c
            w = c["W"][:, c["keep2"]]
            rmat = (c["t"][:, None] * w.T) @ (c["sig"][:, None] * c["V~"][:, c["keep"]].T)
            p, s, vh = np.linalg.svd(rmat, full_matrices=False)
            q = c["qt"][:, c["keep2"]] / c["t"]
            c["U"], c["S"], c["V"] = q @ p, s, vh.T
        elif k == "uout":
            if "U" in self.c:  # end of a core: signs (reading R5), publish
                u, v = o.canonical_signs(self.c["U"], self.c["V"])
                self.out = dict(U=u, S=self.c["S"], V=v)
                self.c = {}
            else:  # the final product of Alg. 6 (U = Q U~[:, :k])
                kk = min(self.k, self.final["S"].size)
                u = self.q_last @ self.final["Ut"][:, :kk]
                self.result = (u, self.final["S"][:kk], self.final["VA"][:, :kk])
        elif k == "alpha":
            qt = self.omega if self.qt is None else self.qt
            self.cur = self.a @ qt
        elif k == "beta":  # local A_p^T Q (the allreduce that follows, if any, sums it)
            self.q_last = self.out["U"]
            self.pending = self.cur = self.a.T @ self.q_last
        elif k == "qt":
            self.qt = self.out["U"]
        elif k == "canon":
            va, ut = self.o.canonical_signs(self.out["U"], self.out["V"])
            self.final = dict(VA=va, S=self.out["S"], Ut=ut)
        else:
            raise AssertionError(f"unknown trace token {tok}")


MIX_SEED = 5


def _replay(rank, world, problem, name, m, n, trace):
    import synth
    from paper_1612_08709_b200 import shard_rows

    if problem in ("tssvd", "tsqr"):
        d = synth.config_inputs(name, m=m)
        omega = None
    else:
        d = synth.config_inputs(name, m=m, n=n)
        omega = d["Omega"]
    r0, r1 = shard_rows(d["A"].shape[0], world, rank)
    rp = Replay(d["A"][r0:r1], omega, lambda w: synth.mixing_params(w, MIX_SEED))
    rp.qt = None
    rp.k = d.get("k", 0)
    for tok in trace:
        rp.run(tok)
    if problem in ("tssvd", "tsqr"):
        res = (rp.out["U"], rp.out["S"], rp.out["V"])
    else:
        res = rp.result
    return res, rp.collectives


def _worker(rank, world, port, problem, name, m, n, out_q):
    sys.path.insert(0, ROOT)
    from paper_1612_08709_b200 import _lib, shard_rows

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth

        cfg = synth.CONFIGS[name]
        mm = m or cfg["m"]
        r0, r1 = shard_rows(mm, world, rank)
        if problem in ("tssvd", "tsqr"):
            trace = _lib.trace(problem, world, r1 - r0, n or cfg["n"], wp=WP)
        else:
            trace = _lib.trace(problem, world, r1 - r0, n, cfg["l"], cfg["iters"], cfg["k"], wp=WP)
        (u, s, v), coll = _replay(rank, world, problem, name, m, n, trace)
        g = torch.from_numpy(np.ascontiguousarray(u.T @ u))
        dist.all_reduce(g)  # orthonormality of the distributed U
        out_q.put((rank, trace, coll, s, v, u, float(np.max(np.abs(g.numpy() - np.eye(g.shape[0]))))))
    finally:
        dist.destroy_process_group()


def _run_world(problem, name, m=None, n=None, world=2):
    port = free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, problem, name, m, n, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def _syncs(trace):
    return [t for t in trace if t.startswith("sync:")]


@pytest.mark.parametrize("name,m,passes_syncs", [("c2", 60_000, 2), ("c1", None, 0)])
def test_two_rank_tssvd_trace_replay(name, m, passes_syncs):
    """tssvd (Alg. 4) on 2 ranks, replayed from the orchestrator's own trace: c2 (w = 100, the
    eigensolver's k and the first discard's r read back: 2 syncs) and c1 (w = 10: every decision
    on the device, no sync before the end)."""
    import oracle
    import synth

    res = _run_world("tssvd", name, m)
    (_, t0, c0, s0, v0, u0, o0), (_, t1, c1, s1, v1, u1, o1) = res
    assert t0 == t1  # equal shards up to one row: identical step sequences
    assert len(_syncs(t0)) == passes_syncs
    whats = [w for w, _ in c0]
    assert whats[0] == "m" and whats.count("gram") == 2 and whats.count("norms") == 2
    assert np.array_equal(s0, s1) and np.array_equal(v0, v1)  # replicated cores agree bitwise
    assert o0 <= 1e-13
    d = synth.config_inputs(name, m=m)
    ref = oracle.tssvd(d["A"], WP, 2)
    assert_tssvd_parity((np.vstack([u0, u1]), s0, v0), ref, passes=2, sigma_tol=1e-12)


def test_two_rank_lowrank_trace_replay():
    """lowrank_svd (Alg. 8) on 2 ranks from the trace: no host round trip before the end,
    the A^T Q allreduce without pad columns (n x even(l)), replicated factors bit-identical,
    and the single-process oracle reproduced."""
    import oracle
    import synth

    m, n = 8_000, 1_001
    res = _run_world("lowrank", "c3", m, n)
    (_, t0, c0, s0, v0, u0, o0), (_, t1, c1, s1, v1, u1, o1) = res
    assert t0 == t1 and _syncs(t0) == [] and t0[-1] == "finish"
    cfg = synth.CONFIGS["c3"]
    betas = [c for w, c in c0 if w == "beta"]
    assert betas == [n * (cfg["l"] + (cfg["l"] & 1))] * (cfg["iters"] + 1)
    assert np.array_equal(s0, s1) and np.array_equal(v0, v1)
    assert o0 <= 1e-13
    d = synth.config_inputs("c3", m=m, n=n)
    ref = oracle.lowrank_svd(d["A"], d["Omega"], cfg["iters"], cfg["k"], WP)
    assert s0.size == ref[1].size == cfg["k"]
    assert_lowrank_parity((np.vstack([u0, u1]), s0, v0), ref, d["A"], d["x0"])


@pytest.mark.parametrize("name,m", [("c2", 60_000), ("c1", None)])
def test_two_rank_tsqr_trace_replay(name, m):
    """tsqr_svd (Alg. 2) on 2 ranks from the orchestrator's trace: each rank's local QR, the R
    factors all-gathered (rank order) and factored again identically, Q_p times its rows of that
    factor (the top of the TSQR tree), discards and the SVD of T = R R~ replicated; no host round
    trip before the end; the single-process oracle (same Omega draws) reproduced."""
    import oracle
    import synth

    res = _run_world("tsqr", name, m)
    (_, t0, c0, s0, v0, u0, o0), (_, t1, c1, s1, v1, u1, o1) = res
    assert t0 == t1 and _syncs(t0) == [] and t0[-1] == "finish"
    n = synth.CONFIGS[name]["n"]
    assert [w for w, _ in c0] == ["m", "allgather", "allgather"]
    assert all(cnt == n * n for w, cnt in c0 if w == "allgather")
    assert np.array_equal(s0, s1) and np.array_equal(v0, v1)
    assert o0 <= 1e-13
    d = synth.config_inputs(name, m=m)
    ref = oracle.tsqr_svd(d["A"], *synth.mixing_params(n, MIX_SEED), WP, 2)
    assert_tssvd_parity((np.vstack([u0, u1]), s0, v0), ref, passes=2, sigma_tol=1e-13)


def test_two_rank_lowrank_tsqr_trace_replay():
    """lowrank_svd_tsqr (Alg. 7) on 2 ranks from the trace: TSQR cores with the R all-gather for
    the row-sharded factors, local TSQR for the replicated n x l ones, the A^T Q allreduce;
    one round trip; the single-process oracle reproduced."""
    import oracle
    import synth

    m, n = 8_000, 1_001
    res = _run_world("lowrank_tsqr", "c3", m, n)
    (_, t0, c0, s0, v0, u0, o0), (_, t1, c1, s1, v1, u1, o1) = res
    assert t0 == t1 and _syncs(t0) == [] and t0[-1] == "finish"
    cfg = synth.CONFIGS["c3"]
    whats = [w for w, _ in c0]
    assert whats.count("allgather") == cfg["iters"] + 2 and whats.count("beta") == cfg["iters"] + 1
    assert np.array_equal(s0, s1) and np.array_equal(v0, v1)
    assert o0 <= 1e-13
    d = synth.config_inputs("c3", m=m, n=n)
    ref = oracle.lowrank_svd_tsqr(d["A"], d["Omega"], cfg["iters"], cfg["k"],
                                  lambda w: synth.mixing_params(w, MIX_SEED), WP)
    assert s0.size == ref[1].size == cfg["k"]
    assert_lowrank_parity((np.vstack([u0, u1]), s0, v0), ref, d["A"], d["x0"])


def test_two_rank_lowrank_lu_trace_replay():
    """lowrank_svd_lu (Alg. 8 with LU-based tracking) on 2 ranks from the trace:
    partial pivoting across the row shards (MAX of the candidates' magnitudes, MIN of the owning
    rank, the pivot row summed from its owner), the replicated n x l eliminations local, one round
    trip; the single-process LU oracle reproduced."""
    import oracle
    import synth

    m, n = 8_000, 1_001
    res = _run_world("lowrank_lu", "c3", m, n)
    (_, t0, c0, s0, v0, u0, o0), (_, t1, c1, s1, v1, u1, o1) = res
    assert t0 == t1 and _syncs(t0) == [] and t0[-1] == "finish"
    cfg = synth.CONFIGS["c3"]
    whats = [w for w, _ in c0]
    assert whats.count("lu_max") == whats.count("lu_owner") == whats.count("lu_row") == cfg["iters"] * cfg["l"]
    assert np.array_equal(s0, s1) and np.array_equal(v0, v1)
    assert o0 <= 1e-13
    d = synth.config_inputs("c3", m=m, n=n)
    ref = oracle.lowrank_svd_lu(d["A"], d["Omega"], cfg["iters"], cfg["k"], WP)
    assert s0.size == ref[1].size == cfg["k"]
    assert_lowrank_parity((np.vstack([u0, u1]), s0, v0), ref, d["A"], d["x0"])


def test_trace_single_rank_has_no_collectives():
    from paper_1612_08709_b200 import _lib

    for t in (_lib.trace("tssvd", 1, 100_000, 100), _lib.trace("lowrank", 1, 10_000, 2_000, 25, 2, 20)):
        assert not [x for x in t if x.startswith("allreduce")]
        assert t[-1] == "finish" or t[-1].startswith("d2h")


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


def test_bench_device_built_inputs_shard_consistently():
    """bench.py's device-built inputs (c5: A does not fit the host) at a reduced size, on the CPU
    generator: two ranks' shards stacked have the prescribed spectrum sigma_j = exp(-(j-1)/15)
    (U_r blocks Q_p / sqrt(P): orthonormal across ranks) above the noise floor, and Omega is the
    same on every rank."""
    sys.path.insert(0, ROOT)
    import bench
    import synth

    cfg = dict(synth.CONFIGS["c5"])
    cfg.update(m=3_000, n=400)
    dev = torch.device("cpu")
    a0, om0 = bench.device_lowrank_inputs(cfg, 0, 1_500, 2, 0, dev)
    a1, om1 = bench.device_lowrank_inputs(cfg, 1_500, 3_000, 2, 1, dev)
    assert torch.equal(om0, om1) and om0.shape == (400, cfg["l"])
    s = np.linalg.svd(torch.cat([a0, a1]).numpy(), compute_uv=False)
    want = synth.spectrum("exp15", cfg["r"])
    # the noise 1e-8 G / sqrt(n) has spectral norm ~1e-8 (sqrt(m / n) + 1) ~ 4e-8
    assert np.max(np.abs(s[:cfg["r"]] - want)) <= 1e-7
    assert s[cfg["r"]] <= 1e-7
    # one rank alone (P = 1): U_r is Haar, same spectrum
    a, _ = bench.device_lowrank_inputs(cfg, 0, 3_000, 1, 0, dev)
    s1 = np.linalg.svd(a.numpy(), compute_uv=False)
    assert np.max(np.abs(s1[:cfg["r"]] - want)) <= 1e-7
