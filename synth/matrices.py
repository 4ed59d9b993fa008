"""Seeded, counter-based synthetic inputs (no method arithmetic here).

Recipe:

* RNG: numpy's Philox4x32-10 with key = (seed, stream) and counter word 1 =
  row-block index, so every row block is drawn independently of the others
  and of the thread that draws it.  Streams: 1 = U Gaussian, 2 = V Gaussian,
  3 = noise G, 4 = Omega, 5 = power-method start vector x0.
* Haar factors (BASELINE.json configs: "U Haar via QR of seeded Gaussian
  blocks"): Householder QR of each Gaussian row block G_b = Q_b R_b, QR of the
  stacked R_b = Q_top R_top, U = blockdiag(Q_b) Q_top diag(sign(diag R_top)).
  That is exactly the sign-fixed (diag R > 0) Q factor of the whole Gaussian
  matrix, i.e. a Haar-distributed orthonormal basis.
* A = U diag(sigma) V^T (+ noise) formed in float64 row block by row block.
* Paper workloads: U, V discrete cosine transforms
  (orthonormal DCT-II, SPEC.md:412 reading) with the Eq. testS / testSl spectra.

Nothing here computes a Gram matrix, an eigendecomposition or a discard.
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

BLOCK_ROWS = 65536  # rows per generator block (fixed: the bytes depend on it)

STREAM_U, STREAM_V, STREAM_NOISE, STREAM_OMEGA, STREAM_X0 = 1, 2, 3, 4, 5


def _threads() -> int:
    return max(1, min(32, os.cpu_count() or 1))


def normal_block(seed: int, stream: int, block: int, rows: int, cols: int) -> np.ndarray:
    """i.i.d. N(0,1) float64 (rows x cols), C order, from Philox(key=(seed,stream), counter=(0,block,0,0))."""
    bg = np.random.Philox(key=np.array([seed, stream], dtype=np.uint64),
                          counter=np.array([0, block, 0, 0], dtype=np.uint64))
    return np.random.Generator(bg).standard_normal(size=(rows, cols))


def _blocks(m: int, block_rows: int = BLOCK_ROWS):
    nb = max(1, -(-m // block_rows))
    return [(b, b * block_rows, min(m, (b + 1) * block_rows)) for b in range(nb)]


def haar(m: int, n: int, seed: int, stream: int, rows: tuple[int, int] | None = None) -> np.ndarray:
    """Rows [r0, r1) of the sign-fixed Q factor of an m x n seeded Gaussian matrix (m >= n).

    Blocked construction.  Only the requested row range is
    materialised, but the R factors of all blocks are needed for Q_top.
    """
    if m < n:
        raise ValueError("haar needs m >= n")
    r0, r1 = rows if rows is not None else (0, m)
    blocks = _blocks(m)
    need = [b for b in blocks if b[2] > r0 and b[1] < r1]

    def fac(bk, want_q):
        b, s, e = bk
        g = normal_block(seed, stream, b, e - s, n)
        if want_q:
            q, r = np.linalg.qr(g, mode="reduced")
            return q, r
        return None, np.linalg.qr(g, mode="r")

    need_ids = {b[0] for b in need}
    with ThreadPoolExecutor(_threads()) as ex:
        facs = list(ex.map(lambda bk: fac(bk, bk[0] in need_ids), blocks))
    rs = [f[1] for f in facs]
    q_top, r_top = np.linalg.qr(np.vstack(rs), mode="reduced")
    d = np.sign(np.diag(r_top))
    d[d == 0] = 1.0
    q_top = q_top * d[None, :]
    offs = np.cumsum([0] + [r.shape[0] for r in rs])
    out = np.empty((r1 - r0, n))

    def emit(bk):
        b, s, e = bk
        ub = facs[b][0] @ q_top[offs[b]:offs[b + 1]]
        lo, hi = max(s, r0), min(e, r1)
        out[lo - r0:hi - r0] = ub[lo - s:hi - s]

    with ThreadPoolExecutor(_threads()) as ex:
        list(ex.map(emit, need))
    return out


def spectrum(kind: str, count: int, **kw) -> np.ndarray:
    """Singular values sigma_1 >= ... (float64).

    kinds: 'log'   : sigma_j = 10^(-decades*(j-1)/(count-1))  (BASELINE configs c1, c2, c4)
           'dec10' : sigma_j = 10^(-(j-1)/10)                 (c3)
           'exp15' : sigma_j = exp(-(j-1)/15)                  (c5)
           'testS' : sigma_j = exp((j-1)/(count-1) ln 1e-20)
    """
    j = np.arange(count, dtype=np.float64)
    if kind == "log":
        return 10.0 ** (-kw["decades"] * j / (count - 1))
    if kind == "dec10":
        return 10.0 ** (-j / 10.0)
    if kind == "exp15":
        return np.exp(-j / 15.0)
    if kind == "testS":
        return np.exp(j / (count - 1) * math.log(1e-20))
    raise ValueError(kind)


def test_matrix(m: int, n: int, sigma: np.ndarray, seed: int,
                rows: tuple[int, int] | None = None) -> np.ndarray:
    """Rows [r0,r1) of A = U diag(sigma) V^T, U (m x n) and V (n x n) Haar (c1, c2, c4)."""
    u = haar(m, n, seed, STREAM_U, rows)
    v = haar(n, n, seed, STREAM_V)
    w = (sigma[:, None] * v.T)  # diag(sigma) V^T
    out = np.empty_like(u)
    step = BLOCK_ROWS

    def mul(s):
        out[s:s + step] = u[s:s + step] @ w

    with ThreadPoolExecutor(_threads()) as ex:
        list(ex.map(mul, range(0, u.shape[0], step)))
    return np.ascontiguousarray(out)


def lowrank_factors(m: int, n: int, r: int, seed: int, rows=None):
    """Haar U_r (rows of m x r), V_r (n x r) for the low-rank configs (c3, c5)."""
    return haar(m, r, seed, STREAM_U, rows), haar(n, r, seed, STREAM_V)


def lowrank_test_matrix(m: int, n: int, r: int, sigma: np.ndarray, noise: float, seed: int,
                        rows: tuple[int, int] | None = None) -> np.ndarray:
    """Rows [r0,r1) of A = U_r diag(sigma) V_r^T + noise * G / sqrt(n), G iid N(0,1) (c3, c5)."""
    r0, r1 = rows if rows is not None else (0, m)
    u, v = lowrank_factors(m, n, r, seed, (r0, r1))
    w = sigma[:, None] * v.T
    out = np.empty((r1 - r0, n))

    def fill(bk):
        b, s, e = bk
        lo, hi = max(s, r0), min(e, r1)
        if lo >= hi:
            return
        g = normal_block(seed, STREAM_NOISE, b, e - s, n)[lo - s:hi - s]
        out[lo - r0:hi - r0] = u[lo - r0:hi - r0] @ w + (noise / math.sqrt(n)) * g

    with ThreadPoolExecutor(_threads()) as ex:
        list(ex.map(fill, _blocks(m)))
    return out


def dct_columns(m: int, k: int, rows: tuple[int, int] | None = None) -> np.ndarray:
    """First k columns of the m x m orthonormal DCT-II matrix C^T (column j = j-th cosine basis
    vector); rows [r0, r1) only when given (row shards of the paper's matrices)."""
    r0, r1 = rows if rows is not None else (0, m)
    i = np.arange(r0, r1, dtype=np.float64)[:, None]
    j = np.arange(k, dtype=np.float64)[None, :]
    c = np.cos(np.pi * (2.0 * i + 1.0) * j / (2.0 * m)) * math.sqrt(2.0 / m)
    c[:, 0] = 1.0 / math.sqrt(m)
    return c


def paper_test_matrix(m: int, n: int, rows: tuple[int, int] | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Eq. originalmat + testS: A = U Sigma V^*, DCT U, V; returns (A, sigma)."""
    s = spectrum("testS", n)
    w = s[:, None] * dct_columns(n, n).T
    r0, r1 = rows if rows is not None else (0, m)
    out = np.empty((r1 - r0, n))
    step = 65536

    def mul(b0):
        b1 = min(r1, b0 + step)
        out[b0 - r0:b1 - r0] = dct_columns(m, n, (b0, b1)) @ w

    with ThreadPoolExecutor(_threads()) as ex:
        list(ex.map(mul, range(r0, r1, step)))
    return out, s


def paper_lowrank_test_matrix(m: int, n: int, l: int) -> tuple[np.ndarray, np.ndarray]:
    """Eq. originalmat + testSl: only Sigma_jj, j <= l, nonzero."""
    s = spectrum("testS", l)
    a = (dct_columns(m, l) * s[None, :]) @ dct_columns(n, l).T
    return a, s


def devils_staircase(k: int) -> np.ndarray:
    """Singular values of Appendix 'devil', restating its Scala recipe:
    for j = 0..k-1, x = round(j * 8^6 / k) in single precision, the octal digits 1-7 of x
    become binary 1s (octal 0 stays 0), read as a binary number, / 2^6 / (1 - 2^-6); sorted
    descending.  Values are multiples of 1/63 in [0, 1], with many repeats."""
    out = np.empty(k)
    scale = np.float32(8.0 ** 6)
    for j in range(k):
        x = int(np.floor(np.float32(np.float32(j) * scale / np.float32(k)) + np.float32(0.5)))  # Math.round(float)
        bits = "".join("0" if ch == "0" else "1" for ch in format(x, "o"))
        out[j] = int(bits, 2) / 2.0 ** 6 / (1.0 - 2.0 ** -6)
    return np.sort(out)[::-1].copy()


def paper_staircase_matrix(m: int, n: int, rows: tuple[int, int] | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Eq. originalmat with the Devil's-staircase spectrum (k = n):
    A = U Sigma V^*, U and V the DCT factors of Eq. originalmat; returns (A, sigma)."""
    s = devils_staircase(n)
    r0, r1 = rows if rows is not None else (0, m)
    a = (dct_columns(m, n, (r0, r1)) * s[None, :]) @ dct_columns(n, n).T
    return a, s


def mixing_params(n: int, seed: int, stream: int = 6) -> tuple[np.ndarray, np.ndarray]:
    """The random numbers of Omega = D F S D~ F S~ (Remark 'randomness') for width n
    (h = n // 2 complex slots): phases [theta_D (h), theta_D~ (h)] uniform in [0, 2 pi), and
    permutations [S (h), S~ (h)] of 0..h-1 by the Fisher-Yates-Durstenfeld shuffle (the draws of
    the method, passed to both paths as inputs)."""
    h = n // 2
    g = np.random.Generator(np.random.Philox(key=np.array([seed, stream], dtype=np.uint64),
                                             counter=np.array([0, n, 0, 0], dtype=np.uint64)))
    phases = g.uniform(0.0, 2.0 * math.pi, size=2 * h)
    perms = np.empty(2 * h, dtype=np.int32)
    for half in range(2):
        p = np.arange(h, dtype=np.int32)
        for i in range(h - 1, 0, -1):  # Durstenfeld: swap p[i] with p[j], j uniform in [0, i]
            j = int(g.integers(0, i + 1))
            p[i], p[j] = p[j], p[i]
        perms[half * h:(half + 1) * h] = p
    return phases, perms


def omega(n: int, l: int, seed: int) -> np.ndarray:
    """Alg. 5 step 1: n x l i.i.d. centred Gaussian start block, shared by both paths."""
    return normal_block(seed, STREAM_OMEGA, 0, n, l)


def power_start(n: int, seed: int) -> np.ndarray:
    """Start vector of the 20-step power method, shared by both paths."""
    return normal_block(seed, STREAM_X0, 0, n, 1)[:, 0].copy()


# BASELINE.json configs.  'm'/'n' are the full sizes; tests scale m (and n for
# low-rank) down with the same recipe for the CPU oracle.
CONFIGS = {
    "c1": dict(kind="tssvd", m=4000, n=10, spec=("log", 6.0), seed=1, passes=2),
    "c2": dict(kind="tssvd", m=2_000_000, n=100, spec=("log", 10.0), seed=2, passes=2),
    "c3": dict(kind="lowrank", m=200_000, n=20_000, r=50, spec=("dec10",), noise=1e-6,
               k=20, l=25, iters=2, seed=3),
    "c4": dict(kind="tssvd", m=8_000_000, n=200, spec=("log", 12.0), seed=4, passes=2),
    "c5": dict(kind="lowrank", m=500_000, n=40_000, r=100, spec=("exp15",), noise=1e-8,
               k=50, l=60, iters=4, seed=5),
    # the paper's own tall-skinny workloads: Eq. originalmat with DCT
    # factors, n = 2000; t3/t4/t5 = Tables 3/4/5 (testS spectrum, Alg. 4 at the reading-Q1
    # wp = 1e-12), s21 = Table 21 (Devil's staircase, wp = 1e-11)
    "t3": dict(kind="tssvd", m=1_000_000, n=2_000, spec=("testS",), gen="dct", seed=0, passes=2, wp=1e-12),
    "t4": dict(kind="tssvd", m=100_000, n=2_000, spec=("testS",), gen="dct", seed=0, passes=2, wp=1e-12),
    "t5": dict(kind="tssvd", m=10_000, n=2_000, spec=("testS",), gen="dct", seed=0, passes=2, wp=1e-12),
    "s21": dict(kind="tssvd", m=10_000, n=2_000, spec=("staircase",), gen="dct", seed=0, passes=2, wp=1e-11),
}


def config_sigma(cfg: dict) -> np.ndarray:
    kind = cfg["spec"][0]
    count = cfg["n"] if cfg["kind"] == "tssvd" else cfg["r"]
    if kind == "log":
        return spectrum("log", count, decades=cfg["spec"][1])
    return spectrum(kind, count)


def config_inputs(name: str, m: int | None = None, n: int | None = None,
                  rows: tuple[int, int] | None = None) -> dict:
    """Host inputs of config `name` (optionally with m / n scaled down, or a row range).

    Returns dict(A=..., sigma=..., plus Omega/x0/k/l/iters for low-rank).
    """
    cfg = dict(CONFIGS[name])
    mm = m or cfg["m"]
    nn = n or cfg["n"]
    out = dict(name=name, m=mm, n=nn, cfg=cfg)
    if cfg.get("gen") == "dct":  # the paper's DCT-factor matrices
        fn = paper_staircase_matrix if cfg["spec"][0] == "staircase" else paper_test_matrix
        out["A"], out["sigma"] = fn(mm, nn, rows)
    elif cfg["kind"] == "tssvd":
        sig = config_sigma(dict(cfg, n=nn))
        out["sigma"] = sig
        out["A"] = test_matrix(mm, nn, sig, cfg["seed"], rows)
    else:
        sig = config_sigma(cfg)
        out["sigma"] = sig
        out["A"] = lowrank_test_matrix(mm, nn, cfg["r"], sig, cfg["noise"], cfg["seed"], rows)
        out["Omega"] = omega(nn, cfg["l"], cfg["seed"])
        out.update(k=cfg["k"], l=cfg["l"], iters=cfg["iters"])
    out["x0"] = power_start(nn, cfg["seed"])
    return out
