"""Parity helpers: compare the CUDA path's factors with the oracle's (SURVEY 8(c) contract)."""
import numpy as np

import oracle

EPS = np.finfo(np.float64).eps


def col_dist(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Per-column sign-invariant distance min(||a_j - b_j||, ||a_j + b_j||)."""
    return np.minimum(np.linalg.norm(a - b, axis=0), np.linalg.norm(a + b, axis=0))


def assert_tssvd_parity(gpu, ref, *, passes: int, sigma_tol: float = 1e-10, uv_const: float = 1e3,
                        ortho_tol: float = 1e-13, parts: int = 1, check_u: bool = True):
    """gpu / ref = (U, sigma, V) as numpy arrays.  Bounds (SURVEY 8(c) parity contract):
    equal kept rank; |d sigma_j| <= sigma_tol * sigma_1; orthonormality after pass 2
    <= ortho_tol on each side; columns within uv_const * eps * (sigma_1 / sigma_j)^2 (reading Q11)."""
    ug, sg, vg = gpu
    ur, sr, vr = ref
    assert sg.size == sr.size, f"kept rank differs: gpu {sg.size} vs oracle {sr.size}"
    if sr.size == 0:
        return {}
    s1 = sr[0]
    ds = np.max(np.abs(sg - sr))
    assert ds <= sigma_tol * s1, f"max |d sigma| = {ds:.3e} > {sigma_tol:g} sigma_1"
    assert np.all(np.diff(sg) <= 0), "sigma not descending"
    out = dict(dsigma=float(ds / s1))
    out["ortho_v_gpu"] = oracle.ortho_error(vg)
    assert out["ortho_v_gpu"] <= ortho_tol, out
    if check_u:
        out["ortho_u_gpu"] = oracle.ortho_error(ug, parts)
        out["ortho_u_ref"] = oracle.ortho_error(ur, parts)
        if passes == 2:
            assert out["ortho_u_gpu"] <= ortho_tol, out
    bound = uv_const * EPS * (s1 / sr) ** 2
    dv = col_dist(vg, vr)
    assert np.all(dv <= bound), f"V columns differ: {dv / bound}"
    out["dv_rel_max"] = float(np.max(dv / bound))
    if check_u:
        du = col_dist(ug, ur)
        assert np.all(du <= bound), f"U columns differ: {du / bound}"
        out["du_rel_max"] = float(np.max(du / bound))
    return out


def assert_lowrank_parity(gpu, ref, a, x0, *, uv_const: float = 1e3, ortho_tol: float = 1e-13):
    """Low-rank (Alg. 8) contract: equal rank; |d sigma_j| <= 1e-10 sigma_1;
    U and V orthonormal to 1e-13; U and V columns sign-invariantly within the Q11 bound
    uv_const * eps * (sigma_1 / sigma_j)^2; spectral error (20 power iterations from the
    shared x0, the same host estimator on both factor sets) within 1% of the oracle's."""
    ug, sg, vg = gpu
    ur, sr, vr = ref
    assert sg.size == sr.size, f"rank differs: gpu {sg.size} vs oracle {sr.size}"
    s1 = sr[0]
    ds = float(np.max(np.abs(sg - sr)))
    assert ds <= 1e-10 * s1, f"max |d sigma| = {ds:.3e}"
    assert np.all(np.diff(sg) <= 0), "sigma not descending"
    out = dict(dsigma=ds / s1, ortho_u=oracle.ortho_error(ug), ortho_v=oracle.ortho_error(vg))
    assert out["ortho_u"] <= ortho_tol and out["ortho_v"] <= ortho_tol, out
    bound = uv_const * EPS * (s1 / sr) ** 2
    dv, du = col_dist(vg, vr), col_dist(ug, ur)
    out["dv_rel_max"] = float(np.max(dv / bound))
    out["du_rel_max"] = float(np.max(du / bound))
    assert np.all(dv <= bound), f"V columns differ: {dv / bound}"
    assert np.all(du <= bound), f"U columns differ: {du / bound}"
    eg = oracle.spectral_error(a, *gpu, x0)
    er = oracle.spectral_error(a, *ref, x0)
    out["spectral_error_gpu"], out["spectral_error_ref"] = eg, er
    assert abs(eg - er) <= 0.01 * er, out
    return out


def assert_grouped_parity(gpu, ref, *, sigma_tol: float = 1e-10, ortho_tol: float = 1e-13, gap: float = 1e-8):
    """Repeated singular values (the Devil's staircase, reading Q4): singular vectors are unique
    only up to a rotation inside each group of equal sigma, so compare the SUBSPACES: for every
    group (consecutive sigma_j within gap * sigma_1), the principal angles between the GPU's and the
    oracle's column spaces (U and V alike) must be ~0 (sines <= 1e-11), besides sigma and
    orthonormality as in assert_tssvd_parity."""
    ug, sg, vg = gpu
    ur, sr, vr = ref
    assert sg.size == sr.size, f"kept rank differs: gpu {sg.size} vs oracle {sr.size}"
    s1 = sr[0]
    assert np.max(np.abs(sg - sr)) <= sigma_tol * s1
    out = dict(ortho_u=oracle.ortho_error(ug), ortho_v=oracle.ortho_error(vg))
    assert out["ortho_u"] <= ortho_tol and out["ortho_v"] <= ortho_tol, out
    j, worst = 0, 0.0
    while j < sr.size:
        e = j + 1
        while e < sr.size and abs(sr[e] - sr[j]) <= gap * s1:
            e += 1
        for a, b in ((ug, ur), (vg, vr)):
            # sine of the largest principal angle as ||(I - B B^T) A||_2 (no 1 - cos^2
            # cancellation: that form cannot resolve angles below ~1e-7)
            res = a[:, j:e] - b[:, j:e] @ (b[:, j:e].T @ a[:, j:e])
            worst = max(worst, float(np.linalg.norm(res, 2)))
        j = e
    out["max_subspace_sine"] = worst
    assert worst <= 1e-11, out
    return out
