"""GPU tests of the tridiagonal-QL eigensolver (csrc/tridiag_eig.cu) that tssvd() uses for
Alg. 4 step 8 ("Calculate the eigendecomposition Z = W D W^*").  Checked against
LAPACK (oracle.sym_eig) and by the properties the step needs: W orthonormal and W^T Z W diagonal
to ~n eps ||Z||.  Run with `pytest -m gpu` on a B200."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1612_08709_b200 as tk  # noqa: E402
from paper_1612_08709_b200._lib import TssvdError  # noqa: E402

DEV = torch.device("cuda", 0)
EPS = np.finfo(float).eps


def second_pass_gram(m, n, cond_exp=10, wp=1e-11, seed=0):
    """Z = Y^T Y of Alg. 4 built by the oracle's own first pass on a constructed
    spectrum sigma_j = 10^(-cond_exp j/(n-1)): the near-identity, graded matrix the solver sees."""
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = 10.0 ** (-cond_exp * np.arange(n) / max(n - 1, 1))
    a = (u * s) @ v.T
    lam, vt = oracle.sym_eig(oracle.gram(a))
    yt = a @ vt
    sig = np.linalg.norm(yt, axis=0)
    keep = sig >= sig.max() * np.sqrt(wp)
    y = yt[:, keep] / sig[keep]
    return y.T @ y


def check(b, lam, v, tol_const=4.0):
    n = b.shape[0]
    nb = np.max(np.abs(np.linalg.eigvalsh(b)))
    tol = tol_const * n * EPS * max(nb, 1e-300)
    k = int(np.sum(lam > 0))
    vk = v[:, :k]
    assert np.all(np.diff(lam) <= 0)
    assert np.max(np.abs(vk.T @ vk - np.eye(k)), initial=0.0) <= tol_const * n * EPS
    w = vk.T @ b @ vk
    assert np.max(np.abs(w - np.diag(np.diag(w))), initial=0.0) <= tol
    ref = np.sort(np.linalg.eigvalsh(b))[::-1]
    assert np.max(np.abs(lam[:k] - ref[:k]), initial=0.0) <= tol
    assert np.all(v[:, k:] == 0) and np.all(lam[k:] == 0)


@pytest.mark.parametrize("m,n", [(20_000, 55), (20_000, 100), (40_000, 160), (5_000, 25)])
def test_ql_on_second_pass_gram(m, n):
    z = second_pass_gram(m, n)
    assert np.max(np.abs(z - np.eye(z.shape[0]))) < 1e-3  # near the identity, graded
    lam, v, it = tk.sym_eig_ql(torch.from_numpy(z).to(DEV))
    check(z, lam.cpu().numpy(), v.cpu().numpy())
    assert it <= 3 * z.shape[0]  # ~1.3 QL iterations per eigenvalue


@pytest.mark.parametrize("n", [1, 2, 3, 4, 33, 64, 127, 160])
def test_ql_random_psd(n):
    rng = np.random.default_rng(n)
    a = rng.standard_normal((2 * n + 3, n))
    b = a.T @ a
    lam, v, _ = tk.sym_eig_ql(torch.from_numpy(b).to(DEV))
    check(b, lam.cpu().numpy(), v.cpu().numpy())
    d, _ = oracle.sym_eig(b)
    assert np.max(np.abs(lam.cpu().numpy() - d)) <= 4 * n * EPS * d[0]


def test_ql_zero_padded_block_and_multiplicity():
    """Device-side discards pad Z with zero rows/columns past r (reading R15): those directions
    are dropped (k = r); an exactly repeated eigenvalue (the identity block) is resolved."""
    z = second_pass_gram(20_000, 40)
    r = z.shape[0]
    zp = np.zeros((r + 7, r + 7))
    zp[:r, :r] = z
    lam, v, _ = tk.sym_eig_ql(torch.from_numpy(zp).to(DEV))
    lam, v = lam.cpu().numpy(), v.cpu().numpy()
    assert int(np.sum(lam > 0)) == r
    check(zp, lam, v)
    lam2, v2, _ = tk.sym_eig_ql(torch.eye(50, dtype=torch.float64, device=DEV) * 3.0)
    assert np.all(lam2.cpu().numpy() == 3.0)
    v2 = v2.cpu().numpy()
    assert np.max(np.abs(v2.T @ v2 - np.eye(50))) <= 1e-15


def test_ql_errors():
    with pytest.raises(TssvdError, match="ENONFINITE"):
        b = torch.eye(10, dtype=torch.float64, device=DEV)
        b[3, 4] = float("nan")
        tk.sym_eig_ql(b)
    with pytest.raises(TssvdError, match="EINVAL"):
        tk.sym_eig_ql(torch.eye(161, dtype=torch.float64, device=DEV))
    lam, v, _ = tk.sym_eig_ql(torch.zeros((6, 6), dtype=torch.float64, device=DEV))
    assert torch.all(lam == 0) and torch.all(v == 0)


def test_ql_in_tssvd_matches_oracle_c2():
    """End to end: Alg. 4 on c2 (reduced m) meets the parity contract with the Z solve the
    process selected (TSSVD_ZEIG=ql: this kernel; default: Jacobi)."""
    from parity import assert_tssvd_parity

    d = synth.config_inputs("c2", m=200_000)
    u, s, v = tk.tssvd(torch.from_numpy(d["A"]).to(DEV), wp=1e-11, passes=2)
    ref = oracle.tssvd(d["A"], 1e-11, 2)
    assert_tssvd_parity((u.cpu().numpy(), s.cpu().numpy(), v.cpu().numpy()), ref, passes=2)
