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
    bound = uv_const * EPS * (s1 / sr) ** 2 + 1e-14
    dv = col_dist(vg, vr)
    assert np.all(dv <= bound), f"V columns differ: {dv / bound}"
    out["dv_rel_max"] = float(np.max(dv / bound))
    if check_u:
        du = col_dist(ug, ur)
        assert np.all(du <= bound), f"U columns differ: {du / bound}"
        out["du_rel_max"] = float(np.max(du / bound))
    return out
