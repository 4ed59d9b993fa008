"""ORACLE (test infrastructure only) -- plain, slow, obviously-correct CPU float64
implementation of the Gram-based SVD hot path of Li, Kluger & Tygert,
"Algorithms for distributed computation of PCA and SVD" (arXiv 1612.08709).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path (``paper_1612_08709_b200``) and never imports it; the only shared
module is ``synth`` (seeded inputs, no method arithmetic).

Every function follows the paper's pseudocode step by step, in the paper's
order and notation.  Library primitives used as single steps: matrix products
(numpy/BLAS), ``numpy.linalg.eigh`` for "Calculate the eigendecomposition"
(LAPACK dsyevd) and ``numpy.linalg.svd`` for "Calculate the singular value
decomposition" (LAPACK dgesdd).  The paper treats both as black boxes
(SPEC.md "Dense kernels: contract-only").

Citations: ``P:n`` = /root/reference/PAPER.md line n.

Readings of the paper taken here (all listed in DESIGN.md "Readings"):
  R1 working precision wp is an explicit argument, default 1e-11.
  R2 "Form the Gram matrix" of a row-partitioned matrix = per-partition Gram,
     summed in a fixed pairwise tree over partitions, then
     symmetrised (B + B^T)/2.
  R3 eigenvalues clamped at 0 and sorted descending.
  R4 Alg. 3's output is sorted by descending Sigma.
  R5 signs: each (u_j, v_j) flipped so the largest-|.| entry of v_j is positive.
  R6 Alg. 6's SVD of B = Q^T A (l x n) is Alg. 4 applied to B^T (n x l).
  R7 Alg. 8 returns the leading k <= l triplets.
  R21 LU-based tracking: partial row pivoting, stop at the first pivot with
      |pivot_j| <= |pivot_1| wp.
"""
from __future__ import annotations

import numpy as np

DEFAULT_WP = 1e-11  # P:137-139 "the working precision could be 10^-11"


# ---------------------------------------------------------------- helpers --
def split_rows(m: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous row partitions (the 'IndexedRowMatrix' partitions)."""
    parts = max(1, min(parts, max(m, 1)))
    edges = [(m * p) // parts for p in range(parts + 1)]
    return [(edges[p], edges[p + 1]) for p in range(parts)]


def tree_sum(items: list[np.ndarray]) -> np.ndarray:
    """Fixed pairwise (left-balanced) tree reduction: 'merging intermediate results
    through multiple levels of a dependency tree'."""
    if not items:
        raise ValueError("tree_sum of an empty list")
    while len(items) > 1:
        nxt = [items[i] + items[i + 1] for i in range(0, len(items) - 1, 2)]
        if len(items) % 2:
            nxt.append(items[-1])
        items = nxt
    return items[0]


def gram(a: np.ndarray, parts: int = 1) -> np.ndarray:
    """Alg. 3/4 step 1: 'Form the Gram matrix B = A^* A'.

    Per-partition A_p^T A_p, aggregated by tree_sum (reading R2), symmetrised.
    """
    b = tree_sum([a[s:e].T @ a[s:e] for s, e in split_rows(a.shape[0], parts)])
    return 0.5 * (b + b.T)


def column_norms(a: np.ndarray, parts: int = 1) -> np.ndarray:
    """Euclidean norms of the columns (Remark 'normalizing'),
    per-partition sums of squares aggregated by tree_sum."""
    ss = tree_sum([np.sum(a[s:e] * a[s:e], axis=0) for s, e in split_rows(a.shape[0], parts)])
    return np.sqrt(ss)


def sym_eig(b: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """'Calculate the eigendecomposition B = V D V^*'.

    LAPACK via numpy.linalg.eigh; descending order; D clamped to >= 0 (R3).
    """
    if not np.all(np.isfinite(b)):
        raise ValueError("non-finite input to sym_eig")
    d, v = np.linalg.eigh(b)
    order = np.argsort(-d, kind="stable")
    return np.maximum(d[order], 0.0), v[:, order]


def keep_mask(s: np.ndarray, wp: float) -> np.ndarray:
    """Discard rule of Alg. 3 step 5 / Alg. 4 steps 5 and 11:
    'view any entry of Sigma as numerically zero that is less than the greatest entry of
    Sigma times the square root of the working precision'."""
    if s.size == 0 or s.max() <= 0.0:
        return np.zeros(s.shape, dtype=bool)
    return s >= s.max() * np.sqrt(wp)


def canonical_signs(u: np.ndarray, v: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Reading R5: flip (u_j, v_j) so that the largest-magnitude entry of v_j is positive
    (ties -> lowest index).  The paper is silent on signs."""
    u = u.copy()
    v = v.copy()
    for j in range(v.shape[1]):
        i = int(np.argmax(np.abs(v[:, j])))
        if v[i, j] < 0:
            v[:, j] = -v[:, j]
            u[:, j] = -u[:, j]
    return u, v


def _check(a: np.ndarray, wp: float) -> None:
    if a.ndim != 2:
        raise ValueError("A must be 2-D")
    if not (0.0 < wp < 1.0):
        raise ValueError("working precision must lie in (0, 1)")
    if a.shape[0] < a.shape[1]:
        raise ValueError("tall-skinny SVD needs m >= n (P:98-104)")
    if not np.all(np.isfinite(a)):
        raise ValueError("non-finite entry in A")


# ------------------------------------------------------------ Algorithm 3 --
def alg3(a: np.ndarray, wp: float = DEFAULT_WP, parts: int = 1):
    """Algorithm 3: Gram-based SVD of a tall and skinny matrix.

    Returns U (m x r), sigma (r, descending), V (n x r).
    """
    _check(a, wp)
    m, n = a.shape
    # Step 1: Form the Gram matrix B = A^* A.
    b = gram(a, parts)
    # Step 2: eigendecomposition B = V D V^*.
    _, v = sym_eig(b)
    # Step 3: Form U~ = A V.
    ut = a @ v
    # Step 4: Sigma = Euclidean norms of the columns of U~ (Remark 'normalizing').
    sig = column_norms(ut, parts)
    # Step 5: discard entries of Sigma below max(Sigma) * sqrt(wp), with the
    # corresponding columns of U~ and V.
    keep = keep_mask(sig, wp)
    sig, ut, v = sig[keep], ut[:, keep], v[:, keep]
    # Step 6: Form U = U~ Sigma^{-1}.
    u = ut / sig[None, :] if sig.size else ut
    # Reading R4: descending Sigma.
    order = np.argsort(-sig, kind="stable")
    return u[:, order], sig[order], v[:, order]


# ------------------------------------------------------------ Algorithm 4 --
def alg4(a: np.ndarray, wp: float = DEFAULT_WP, parts: int = 1, return_pass1: bool = False):
    """Algorithm 4: Gram-based SVD with double orthonormalization.

    Returns U (m x r'), sigma (r', descending), V (n x r') [, Y after pass 1].
    """
    _check(a, wp)
    m, n = a.shape
    # Step 1: B = A^* A.
    b = gram(a, parts)
    # Step 2: B = V~ D~ V~^*.
    _, vt = sym_eig(b)
    # Step 3: Y~ = A V~.
    yt = a @ vt
    # Step 4: Sigma~ = column norms of Y~.
    st = column_norms(yt, parts)
    # Step 5: discard below max(Sigma~) sqrt(wp).
    keep = keep_mask(st, wp)
    st, yt, vt = st[keep], yt[:, keep], vt[:, keep]
    r = st.size
    if r == 0:
        z = np.zeros((m, 0)), np.zeros(0), np.zeros((n, 0))
        return (*z, np.zeros((m, 0))) if return_pass1 else z
    # Step 6: Y = Y~ Sigma~^{-1}.
    y = yt / st[None, :]
    # Step 7: Z = Y^* Y.
    z = gram(y, parts)
    # Step 8: Z = W D W^*.
    _, w = sym_eig(z)
    # Step 9: Q~ = Y W.
    qt = y @ w
    # Step 10: T = column norms of Q~.
    t = column_norms(qt, parts)
    # Step 11: discard below max(T) sqrt(wp), with columns of Q~ and W.
    keep2 = keep_mask(t, wp)
    t, qt, w = t[keep2], qt[:, keep2], w[:, keep2]
    # Step 12: Q = Q~ T^{-1}.
    q = qt / t[None, :]
    # Step 13: R = T W^* Sigma~ V~^*   (r' x n).
    rmat = (t[:, None] * w.T) @ (st[:, None] * vt.T)
    # Step 14: SVD R = P Sigma V^*.
    p, sig, vh = np.linalg.svd(rmat, full_matrices=False)
    # Step 15: U = Q P.
    u = q @ p
    out = (u, sig, vh.T)
    return (*out, y) if return_pass1 else out


def tssvd(a: np.ndarray, wp: float = DEFAULT_WP, passes: int = 2, parts: int = 1):
    """Problem {1}: Alg. 4 (passes=2) or Alg. 3 (passes=1), canonical signs (R5)."""
    if passes not in (1, 2):
        raise ValueError("passes must be 1 or 2")
    u, s, v = (alg4 if passes == 2 else alg3)(a, wp, parts)
    u, v = canonical_signs(u, v)
    return u, s, v


# ------------------------------------------------------- Algorithms 5,6,8 --
def subspace_iteration(a: np.ndarray, omega: np.ndarray, i: int, wp: float = DEFAULT_WP,
                       parts: int = 1) -> np.ndarray:
    """Algorithm 5 with Alg. 3 inside and Alg. 4 in the last step (Alg. 8).

    'we use Q = U and R = Sigma V^*': the orthonormal factor of each
    tall-skinny factorization is the U returned by Alg. 3 / Alg. 4.
    """
    m, n = a.shape
    l = omega.shape[1]
    if not (0 < l < min(m, n)) or i < 0:
        raise ValueError("need 0 < l < min(m, n) and i >= 0 (P:705-707)")
    # Step 1: Q~_0 = n x l Gaussian (supplied by the caller, shared by both paths).
    qt = omega
    for _ in range(i):
        # Step 3: Y_j = A Q~_{j-1}.
        y = a @ qt
        # Step 4: Y_j = Q_j R_j via Alg. 3.
        q, _, _ = alg3(y, wp, parts)
        # Step 5: Y~_j = A^* Q_j  (rows aggregated over partitions, tree order).
        yt = tree_sum([a[s:e].T @ q[s:e] for s, e in split_rows(m, parts)])
        # Step 6: Y~_j = Q~_j R~_j via Alg. 3.
        qt, _, _ = alg3(yt, wp, 1)
    # Step 8: Y = A Q~_i.
    y = a @ qt
    # Step 9: Y = Q R with double orthonormalization (Alg. 4).
    q, _, _ = alg4(y, wp, parts)
    return q


def direct_svd(a: np.ndarray, q: np.ndarray, wp: float = DEFAULT_WP, parts: int = 1):
    """Algorithm 6.  Reading R6: the SVD of B is Alg. 4 on B^T = A^* Q."""
    m, n = a.shape
    # Step 1: B = Q^* A, formed as B^T = A^* Q (rows aggregated over partitions).
    bt = tree_sum([a[s:e].T @ q[s:e] for s, e in split_rows(m, parts)])
    # Step 2: B = U~ Sigma V^*  <=>  B^T = V Sigma U~^*.
    v, sig, ut = alg4(bt, wp, 1)
    # Step 3: U = Q U~.
    u = q @ ut
    return u, sig, v


def lowrank_svd(a: np.ndarray, omega: np.ndarray, i: int, k: int | None = None,
                wp: float = DEFAULT_WP, parts: int = 1):
    """Algorithm 8 = Alg. 6 fed with Alg. 5 using Alg. 3 and Alg. 4.

    Returns the leading k triplets (reading R7), canonical signs (R5).
    """
    l = omega.shape[1]
    k = l if k is None else k
    if not (0 < k <= l):
        raise ValueError("need 0 < k <= l")
    q = subspace_iteration(a, omega, i, wp, parts)
    u, s, v = direct_svd(a, q, wp, parts)
    kk = min(k, s.size)
    u, v = canonical_signs(u[:, :kk], v[:, :kk])
    return u, s[:kk], v


# ------------------------------------------- Algorithms 1, 2, 7 (TSQR) --
def mix_rows(a: np.ndarray, phases: np.ndarray, perms: np.ndarray, inverse: bool = False) -> np.ndarray:
    """Remark 'randomness': Omega = D F S D~ F S~ applied to every row of A (every
    column of A^*), the real rows viewed as h = n // 2 complex numbers (pairs (x_2k, x_2k+1) =
    real and imaginary parts).  phases = [theta_D (h), theta_D~ (h)] (D = diag(exp(i theta)));
    perms = [S (h), S~ (h)] with (S z)_k = z_{S[k]}; F = the unitary DFT of length h.  Reading
    R17: for odd n the last real entry is left unmixed.  inverse=True applies Omega^{-1} = Omega^*.
    """
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[1]
    h = n // 2
    out = a.copy()
    if h == 0:  # n = 1: the single coordinate is the unmixed last one (reading R17)
        return out
    z = a[:, 0:2 * h:2] + 1j * a[:, 1:2 * h:2]
    d1, d2 = np.exp(1j * phases[:h]), np.exp(1j * phases[h:2 * h])
    s1, s2 = perms[:h].astype(np.int64), perms[h:2 * h].astype(np.int64)
    if not inverse:  # z <- D F S D~ F S~ z  (rightmost first)
        z = z[:, s2]
        z = np.fft.fft(z, axis=1, norm="ortho")
        z = z * d2[None, :]
        z = z[:, s1]
        z = np.fft.fft(z, axis=1, norm="ortho")
        z = z * d1[None, :]
    else:  # z <- S~^-1 F^* D~^* S^-1 F^* D^* z
        z = z * np.conj(d1)[None, :]
        z = np.fft.ifft(z, axis=1, norm="ortho")
        w = np.empty_like(z)
        w[:, s1] = z
        z = w * np.conj(d2)[None, :]
        z = np.fft.ifft(z, axis=1, norm="ortho")
        w = np.empty_like(z)
        w[:, s2] = z
        z = w
    out[:, 0:2 * h:2] = z.real
    out[:, 1:2 * h:2] = z.imag
    return out


def r_keep(r: np.ndarray, wp: float) -> np.ndarray:
    """Alg. 1 step 3 / Alg. 2 steps 3, 5: 'view any diagonal
    entry of R as numerically zero that is less than the first diagonal entry of R times the
    working precision' (magnitudes: R's diagonal signs are a convention of the QR)."""
    d = np.abs(np.diag(r))
    if d.size == 0 or d[0] == 0.0:
        return np.zeros(d.shape, dtype=bool)
    return d >= d[0] * wp


def alg1(a: np.ndarray, phases: np.ndarray, perms: np.ndarray, wp: float = DEFAULT_WP):
    """Algorithm 1: randomized TSQR-based SVD of a tall-skinny matrix.
    'Using the TSQR method compute B^* = Q R' is a QR factorization (TSQR is how the paper
    distributes it; the factorization is unique up to the signs of R's rows): LAPACK's
    Householder QR here.  Returns U (m x r), sigma (r, descending), V (n x r)."""
    _check(a, wp)
    # Step 1: B = Omega A^*, i.e. B^* = A Omega^* = every row of A mixed.
    bs = mix_rows(a, phases, perms)
    # Step 2: B^* = Q R.
    q, r = np.linalg.qr(bs, mode="reduced")
    # Step 3: discard rows of R with numerically zero diagonal, columns of Q.
    keep = r_keep(r, wp)
    q, r = q[:, keep], r[keep, :]
    # Step 4: R = U~ Sigma V~^*.
    ut, sig, vth = np.linalg.svd(r, full_matrices=False)
    # Step 5: U = Q U~.  Step 6: V = Omega^{-1} V~.
    u = q @ ut
    v = mix_rows(vth, phases, perms, inverse=True).T
    return u, sig, v


def alg2(a: np.ndarray, phases: np.ndarray, perms: np.ndarray, wp: float = DEFAULT_WP):
    """Algorithm 2: Algorithm 1 with double orthonormalization."""
    _check(a, wp)
    # Step 1: B^* = every row of A mixed.
    bs = mix_rows(a, phases, perms)
    # Step 2: B^* = Q~ R~.  Step 3: discard.
    qt, rt = np.linalg.qr(bs, mode="reduced")
    keep = r_keep(rt, wp)
    qt, rt = qt[:, keep], rt[keep, :]
    # Step 4: Q~ = Q R.  Step 5: discard.
    q, r = np.linalg.qr(qt, mode="reduced")
    keep2 = r_keep(r, wp)
    q, r = q[:, keep2], r[keep2, :]
    # Step 6: T = R R~.  Step 7: T = U~ Sigma V~^*.
    t = r @ rt
    ut, sig, vth = np.linalg.svd(t, full_matrices=False)
    # Step 8: U = Q U~.  Step 9: V = Omega^{-1} V~.
    u = q @ ut
    v = mix_rows(vth, phases, perms, inverse=True).T
    return u, sig, v


def tsqr_svd(a: np.ndarray, phases: np.ndarray, perms: np.ndarray, wp: float = DEFAULT_WP, passes: int = 2):
    """Problem {1} by Alg. 2 (passes=2) or Alg. 1 (passes=1), canonical signs (R5)."""
    u, s, v = (alg2 if passes == 2 else alg1)(a, phases, perms, wp)
    return canonical_signs(u, v)[0], s, canonical_signs(u, v)[1]


def lowrank_svd_tsqr(a: np.ndarray, omega: np.ndarray, i: int, k: int | None, mixes,
                     wp: float = DEFAULT_WP):
    """Algorithm 7 = Alg. 6 fed with Alg. 5 using Alg. 1 (steps 4, 6) and Alg. 2
    (the last step); reading R6: Alg. 6's SVD of B is Alg. 2 on B^T.  mixes(width) returns the
    (phases, perms) of the random orthogonal matrix for a width-`width` factorization (each
    factorization's own Omega; seeded by the caller, shared with the CUDA path)."""
    m, n = a.shape
    l = omega.shape[1]
    k = l if k is None else k
    qt = omega
    for _ in range(i):
        y = a @ qt
        q, _, _ = alg1(y, *mixes(y.shape[1]), wp)
        yt = a.T @ q
        qt, _, _ = alg1(yt, *mixes(yt.shape[1]), wp)
    y = a @ qt
    q, _, _ = alg2(y, *mixes(y.shape[1]), wp)
    bt = a.T @ q
    v, sig, ut = alg2(bt, *mixes(bt.shape[1]), wp)
    u = q @ ut
    kk = min(k, sig.size)
    u, v = canonical_signs(u[:, :kk], v[:, :kk])
    return u, sig[:kk], v


# ---------------------------------------- LU-based subspace tracking --
def lu_tracking_factor(y: np.ndarray, wp: float = DEFAULT_WP):
    """in the intermediate steps of Alg. 5 'replacing Q with the lower
    triangular/trapezoidal factor L in an LU factorization is sufficient ... the column space of L
    is the same as the column space of Q'.  Gaussian elimination with partial (row) pivoting of
    the tall Y, column by column: the pivot of column j is its largest-|.| entry among the rows
    not yet chosen (ties: the lowest row index); the multipliers y_ij / pivot form column j of L;
    the remaining columns lose the multiple of the pivot row.  Returned L is Y's row order (the
    P L of Y = P L U): 1 at each pivot row's own column, 0 right of it.  Reading R21: elimination
    stops at the first numerically zero pivot, |pivot_j| <= |pivot_1| wp (the Alg. 1 rule,
    P:534-538); the r columns before it are returned."""
    w = np.array(y, dtype=np.float64, copy=True)
    m, l = w.shape
    lmat = np.zeros((m, l))
    chosen = np.zeros(m, dtype=bool)
    p1 = 0.0
    r = 0
    for j in range(l):
        mag = np.abs(w[:, j])
        mag[chosen] = -1.0
        p = int(np.argmax(mag))
        pv = w[p, j]
        if j == 0:
            p1 = abs(pv)
        if not (p1 > 0.0 and abs(pv) > p1 * wp):
            break
        mult = w[:, j] / pv
        mult[chosen] = 0.0
        mult[p] = 1.0
        lmat[:, j] = mult
        urow = w[p, j + 1:].copy()
        w[:, j + 1:] -= np.outer(mult, urow)
        chosen[p] = True
        r = j + 1
    return lmat[:, :r], r


def lowrank_svd_lu(a: np.ndarray, omega: np.ndarray, i: int, k: int | None = None,
                   wp: float = DEFAULT_WP):
    """Alg. 8 with LU-based subspace tracking: Alg. 5's steps 4 and 6
    take the L factor of Y_j / Y~_j (lu_tracking_factor) instead of Alg. 3's Q; the last step
    (Alg. 4) and Alg. 6 are unchanged.  The column spaces are those of Alg. 8, so in exact
    arithmetic the result is Alg. 8's."""
    l = omega.shape[1]
    k = l if k is None else k
    qt = omega
    for _ in range(i):
        # Step 3, step 4 with L
        q, _ = lu_tracking_factor(a @ qt, wp)
        # Step 5, step 6 with L
        qt, _ = lu_tracking_factor(a.T @ q, wp)
    # Step 8, step 9: Alg. 4
    q, _, _ = alg4(a @ qt, wp)
    u, s, v = direct_svd(a, q, wp)
    kk = min(k, s.size)
    u, v = canonical_signs(u[:, :kk], v[:, :kk])
    return u, s[:kk], v
