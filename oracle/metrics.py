"""ORACLE (test infrastructure only) -- accuracy measures of the paper's tables.

Table 'heads': ||A - U Sigma V^*||_2 estimated by 20 power iterations
 and max|U^* U - I|, max|V^* V - I|.  Used on the oracle's AND the
CUDA path's factors alike (same start vector x0 from ``synth.power_start``).
"""
from __future__ import annotations

import numpy as np

from .gram_svd import gram


def spectral_error(a: np.ndarray, u: np.ndarray, s: np.ndarray, v: np.ndarray,
                   x0: np.ndarray, iters: int = 20) -> float:
    """||A - U diag(s) V^T||_2 by `iters` power iterations on M^T M.

    x <- M^T (M x) / ||.||, M never materialised (Mx = Ax - U(s * (V^T x))); returns ||M x_iters||.
    """
    def mv(x):
        return a @ x - u @ (s * (v.T @ x))

    def mtv(y):
        return a.T @ y - v @ (s * (u.T @ y))

    x = x0 / np.linalg.norm(x0)
    for _ in range(iters):
        x = mtv(mv(x))
        nx = np.linalg.norm(x)
        if nx == 0.0:
            return 0.0
        x = x / nx
    return float(np.linalg.norm(mv(x)))


def ortho_error(u: np.ndarray, parts: int = 1) -> float:
    """max |U^* U - I|, U^* U formed like the Gram of step 1 (partition tree)."""
    if u.shape[1] == 0:
        return 0.0
    return float(np.max(np.abs(gram(u, parts) - np.eye(u.shape[1]))))
