"""GPU parity of the TSQR-based Algorithms 1, 2 (tsqr_svd) and 7 (lowrank_svd_tsqr) against the
oracle (oracle.tsqr_svd / oracle.lowrank_svd_tsqr) on the same seeded inputs and the same random
draws of Omega = D F S D~ F S~ (synth.mixing_params).  Run with `pytest -m gpu` on a B200."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from parity import assert_lowrank_parity, assert_tssvd_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1612_08709_b200 as tk  # noqa: E402
from paper_1612_08709_b200._lib import TssvdError  # noqa: E402

DEV = torch.device("cuda", 0)
PAPER = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
EPS = np.finfo(np.float64).eps


def to_dev(a):
    """Device copy with an even leading dimension (odd widths: one pad column, [:, :n] view)."""
    a = np.ascontiguousarray(a)
    if a.shape[1] & 1:
        buf = torch.zeros((a.shape[0], a.shape[1] + 1), dtype=torch.float64, device=DEV)
        buf[:, :a.shape[1]] = torch.from_numpy(a).to(DEV)
        return buf[:, :a.shape[1]]
    return torch.from_numpy(a).to(DEV)


def draws(n, seed):
    ph, pm = synth.mixing_params(n, seed)
    return ph, pm, torch.from_numpy(ph).to(DEV), torch.from_numpy(pm).to(DEV)


def run(a, passes, seed=1, wp=1e-11):
    ph, pm, dph, dpm = draws(a.shape[1], seed)
    u, s, v = tk.tsqr_svd(to_dev(a), dph, dpm, wp=wp, passes=passes)
    torch.cuda.synchronize()
    gpu = (u.cpu().numpy(), s.cpu().numpy(), v.cpu().numpy())
    ref = oracle.tsqr_svd(a, ph, pm, wp, passes)
    return gpu, ref


# QR-based: no squaring of the condition number -- sigma to 1e-13 sigma_1, U and V orthonormal to
# 1e-13 after either algorithm, columns within uv_const eps (sigma_1 / sigma_j)^2 (the Q11 form,
# loose here).
@pytest.mark.parametrize("passes", [1, 2])
@pytest.mark.parametrize("m,n", [(1, 1), (2, 2), (37, 10), (192, 100), (193, 100), (385, 100), (5000, 26),
                                 (256, 64), (257, 64), (65, 65), (300_001, 66),
                                 (12_345, 33), (100_003, 100), (70_001, 128), (50_000, 127), (3, 3)])
def test_tsqr_svd_random(m, n, passes):
    """Several leaf blocks and tree levels with ragged tails (the leaf block is 192 rows for
    n > 64, 256 for n <= 64: 193 / 257 leave a one-row block), odd widths (reading R17), a single
    row, both leaf shapes around n = 64."""
    rng = np.random.default_rng(m * 7 + n)
    a = rng.standard_normal((m, n)) * np.exp(-np.arange(n) / max(n, 1) * 6)[None, :]
    gpu, ref = run(a, passes)
    out = assert_tssvd_parity(gpu, ref, passes=2, sigma_tol=1e-13)
    assert out["ortho_u_gpu"] <= 1e-13


@pytest.mark.parametrize("cfg", ["c1", "c2"])
@pytest.mark.parametrize("passes", [1, 2])
def test_tsqr_svd_configs(cfg, passes):
    """BASELINE configs c1 (4000 x 10) and c2 (2e6 x 100, at full size): the constructed spectra
    (log-spaced to 1e-6 / 1e-10); sigma against the oracle and the true singular values."""
    d = synth.config_inputs(cfg)
    gpu, ref = run(d["A"], passes, seed=2)
    assert_tssvd_parity(gpu, ref, passes=2, sigma_tol=1e-13)
    assert np.max(np.abs(gpu[1] - d["sigma"])) <= 1e-13 * d["sigma"][0]


@pytest.mark.parametrize("passes", [1, 2])
def test_tsqr_svd_rank_deficient(passes):
    """Discards (Alg. 1 step 3, Alg. 2 steps 3 and 5): zero and duplicated columns give
    |R_jj| ~ 0 rows; the kept rank and the surviving triplets match the oracle."""
    rng = np.random.default_rng(5)
    # separated spectrum (1 .. 1e-3) so the per-column comparison is meaningful, then three
    # dependent columns
    u0 = np.linalg.qr(rng.standard_normal((3000, 40)))[0]
    v0 = np.linalg.qr(rng.standard_normal((40, 40)))[0]
    a = (u0 * np.logspace(0, -3, 40)) @ v0.T
    a[:, 7] = 0.0
    a[:, 20] = a[:, 3]
    a[:, 31] = 2 * a[:, 11] - a[:, 5]
    gpu, ref = run(a, passes)
    assert gpu[1].size == ref[1].size == 37
    assert_tssvd_parity(gpu, ref, passes=2, sigma_tol=1e-13)


def test_tsqr_svd_degenerate():
    """A = 0: nothing kept (R_11 = 0); a NaN: TSSVD_ENONFINITE; n > 128 and host tensors refused."""
    ph, pm, dph, dpm = draws(16, 1)
    u, s, v = tk.tsqr_svd(torch.zeros((100, 16), dtype=torch.float64, device=DEV), dph, dpm)
    assert s.numel() == 0
    a = torch.randn((500, 16), dtype=torch.float64, device=DEV)
    a[123, 4] = float("nan")
    with pytest.raises(TssvdError) as e:
        tk.tsqr_svd(a, dph, dpm)
    assert e.value.status == 2
    _, _, dph2, dpm2 = draws(130, 1)
    with pytest.raises(TssvdError) as e:
        tk.tsqr_svd(torch.randn((500, 130), dtype=torch.float64, device=DEV), dph2, dpm2)
    assert e.value.status == 1


def test_tsqr_svd_inplace_and_stats():
    """U may overwrite A (same buffer); the call reports its TSQR passes."""
    rng = np.random.default_rng(9)
    a = rng.standard_normal((20_000, 50)) * np.exp(-np.arange(50) / 50 * 6)[None, :]
    ph, pm, dph, dpm = draws(50, 4)
    A = to_dev(a)
    u, s, v = tk.tsqr_svd(A, dph, dpm, passes=2, inplace=True)
    torch.cuda.synchronize()
    assert u.data_ptr() == A.data_ptr()
    ref = oracle.tsqr_svd(a, ph, pm, 1e-11, 2)
    assert_tssvd_parity((u.cpu().numpy(), s.cpu().numpy(), v.cpu().numpy()), ref, passes=2, sigma_tol=1e-13)
    st = tk.last_stats()
    assert st["ranks"] == [50, 50]


# ------------------------------------------------------------------ Alg. 7 --
def run_lowrank(a, omega, iters, k, seed, wp=1e-11):
    l = omega.shape[1]
    mixes = lambda w: synth.mixing_params(w, seed)  # noqa: E731
    ph, pm = tk.mixing_tables(mixes, l, DEV)
    u, s, v = tk.lowrank_svd_tsqr(to_dev(a), to_dev(omega), iters, ph, pm, k=k, wp=wp)
    torch.cuda.synchronize()
    gpu = (u.cpu().numpy(), s.cpu().numpy(), v.cpu().numpy())
    ref = oracle.lowrank_svd_tsqr(a, omega, iters, k, mixes, wp)
    return gpu, ref


def test_lowrank_tsqr_c3_scaled():
    """c3's spectrum (rank 50, decaying, 1e-6 noise) at 20000 x 2000, l = 25, i = 2, k = 20."""
    d = synth.config_inputs("c3", m=20_000, n=2_000)
    gpu, ref = run_lowrank(d["A"], d["Omega"], d["iters"], d["k"], seed=3)
    assert_lowrank_parity(gpu, ref, d["A"], d["x0"])


@pytest.mark.parametrize("key,l", [("alg7_l20_i2_m1e4_n2000", 20), ("alg7_l10_i2", 10)])
def test_paper_alg7_gpu(key, l):
    """PAPER.md:1039, 1084-1087 (Tables 8 and 10, Algorithm 7) on the GPU path with the recorded
    seeds: the residual is sigma_{r+1} of Eq. testSl (2.64e-12 / 7.74e-12) and equals the
    oracle's; kept ranks 11 / 5 as the oracle's."""
    g = PAPER[key]
    a, sig = synth.paper_lowrank_test_matrix(10_000, 2_000, l)
    seed = g["seed"]
    gpu, ref = run_lowrank(a, synth.omega(2_000, l, seed), g["i"], l, seed)
    assert gpu[1].size == ref[1].size
    x0 = synth.power_start(2_000, 7)
    err = oracle.spectral_error(a, *gpu, x0)
    assert err == pytest.approx(g["spectral_error"], rel=5e-3)
    assert oracle.ortho_error(gpu[0]) <= 1e-14 * 10 and oracle.ortho_error(gpu[2]) <= 1e-14 * 10
    assert np.max(np.abs(gpu[1] - ref[1])) <= 1e-13 * ref[1][0]


def test_lowrank_tsqr_rank_collapse():
    """A of exact rank 6 < l = 16: the first factorization keeps 6, every later one has width 6
    (its Omega drawn for width 6, row 5 of the tables), k = 10 returns 6 triplets."""
    rng = np.random.default_rng(11)
    a = rng.standard_normal((4000, 6)) @ rng.standard_normal((6, 300))
    omega = synth.omega(300, 16, 11)
    gpu, ref = run_lowrank(a, omega, 2, 10, seed=11)
    assert gpu[1].size == ref[1].size == 6
    assert np.max(np.abs(gpu[1] - ref[1])) <= 1e-13 * ref[1][0]
