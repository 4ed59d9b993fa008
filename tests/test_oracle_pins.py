"""Pins of the ORACLE against things other than itself (CPU only, -m "not gpu").

Each pin is chosen so that a plausible mistake in oracle/ (a dropped Sigma^-1,
wp instead of sqrt(wp), a transposed operand, eigenvalues instead of explicit
norms, a missing second pass, a wrong Alg. 5 wiring) fails at least one test:

* closed forms and SPEC.md's [TRIVIAL] examples   (tests/golden/spec_examples.json)
* constructed spectra with known U, sigma, V      (synth: A = U diag(sigma) V^T)
* brute force on tiny inputs (explicit loops; numpy.linalg.svd of A itself)
* values printed in the paper                      (tests/golden/paper_values.json)
* invariants (orthonormality, shard invariance, estimator monotonicity)
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SPEC = json.load(open(os.path.join(GOLD, "spec_examples.json")))
PAPER = json.load(open(os.path.join(GOLD, "paper_values.json")))
EPS = np.finfo(np.float64).eps


def arr(x):
    return np.array(x, dtype=np.float64)


# ------------------------------------------------------------ closed forms --
def test_tree_sum_closed_form():
    e = SPEC["tree_sum_1234"]
    assert oracle.tree_sum([arr([[p]]) for p in e["parts"]])[0, 0] == e["sum"]
    x = arr([[3.0]])
    assert oracle.tree_sum([x]) is x
    with pytest.raises(ValueError):
        oracle.tree_sum([])


def test_tree_sum_vs_sequential_fold():
    rng = np.random.default_rng(0)
    parts = [rng.standard_normal((3, 3)) for _ in range(7)]
    seq = parts[0].copy()
    for p in parts[1:]:
        seq = seq + p
    assert np.max(np.abs(oracle.tree_sum(parts) - seq)) <= 1e-12 * np.max(np.abs(seq))


@pytest.mark.parametrize("key", ["gram_stacked_identity", "gram_ones_column"])
def test_gram_closed_forms(key):
    e = SPEC[key]
    assert np.array_equal(oracle.gram(arr(e["A"])), arr(e["B"]))


def test_gram_brute_force_loops():
    """B_ij = sum_k a_ki a_kj written as explicit loops (tiny input), several partitions."""
    rng = np.random.default_rng(1)
    a = rng.standard_normal((50, 6))
    brute = np.zeros((6, 6))
    for i in range(6):
        for j in range(6):
            brute[i, j] = sum(a[k, i] * a[k, j] for k in range(50))
    for parts in (1, 4, 7):
        b = oracle.gram(a, parts)
        assert np.array_equal(b, b.T)
        assert np.max(np.abs(b - brute)) <= 1e-13 * np.max(np.abs(brute))


def test_column_norms_brute_force():
    rng = np.random.default_rng(2)
    a = rng.standard_normal((37, 5))
    brute = [np.sqrt(sum(a[k, j] ** 2 for k in range(37))) for j in range(5)]
    assert np.allclose(oracle.column_norms(a, 3), brute, rtol=1e-15, atol=0)


def test_sym_eig_closed_forms():
    e = SPEC["eig_diag"]
    d, v = oracle.sym_eig(arr(e["B"]))
    assert np.array_equal(d, arr(e["eigvals"]))
    assert np.array_equal(np.abs(v), arr([[0, 1], [1, 0]]))
    e = SPEC["eig_rank1"]
    d, v = oracle.sym_eig(arr(e["B"]))
    assert np.allclose(d, e["eigvals"], atol=1e-15)
    assert d[1] >= 0.0  # clamp (reading R3)
    assert np.allclose(np.abs(v[:, 0]), e["v1"], atol=1e-15)


def test_sym_eig_invariants_random_psd():
    """B V = V D and V^T V = I (a property independent of how eigh works)."""
    rng = np.random.default_rng(3)
    a = rng.standard_normal((9, 4))
    b = a.T @ a
    d, v = oracle.sym_eig(b)
    assert np.all(np.diff(d) <= 0)
    assert np.max(np.abs(b @ v - v * d[None, :])) <= 1e-13 * d[0]
    assert np.max(np.abs(v.T @ v - np.eye(4))) <= 1e-14
    # eigenvalues of A^T A are the squared singular values of A (textbook identity)
    assert np.allclose(d, np.linalg.svd(a, compute_uv=False) ** 2, rtol=1e-12)


def test_keep_mask_sqrt_wp_rule():
    """threshold is max(Sigma) * sqrt(wp), not max(Sigma) * wp."""
    s = arr([1.0, 3.2e-6, 3.1e-6, 5e-11])
    assert list(oracle.keep_mask(s, 1e-11)) == [True, True, False, False]
    assert list(oracle.keep_mask(s, 1e-22)) == [True, True, True, True]
    assert not oracle.keep_mask(np.zeros(3), 1e-11).any()


def test_spectral_error_closed_form():
    e = SPEC["residual_diag51"]
    a = arr(e["A"])
    u = arr([[1.0], [0.0]])
    v = arr([[1.0], [0.0]])
    est = oracle.spectral_error(a, u, arr([5.0]), v, arr([0.3, 0.7]))
    assert abs(est - e["residual"]) <= 1e-10


def test_spectral_error_known_truncation_and_monotone():
    """Exact rank-r truncation of a known spectrum leaves sigma_{r+1}."""
    d = synth.config_inputs("c1")
    a, s = d["A"], d["sigma"]
    u = synth.haar(4000, 10, 1, synth.matrices.STREAM_U)
    v = synth.haar(10, 10, 1, synth.matrices.STREAM_V)
    est = [oracle.spectral_error(a, u[:, :4], s[:4], v[:, :4], d["x0"], it) for it in (2, 5, 20)]
    assert abs(est[-1] - s[4]) <= 1e-6 * s[4]
    assert est[0] <= est[1] * (1 + 1e-12) <= est[2] * (1 + 1e-12)
    # brute force: the 2-norm of the residual matrix itself
    brute = np.linalg.norm(a - (u[:, :4] * s[:4]) @ v[:, :4].T, 2)
    assert abs(est[-1] - brute) <= 1e-6 * brute


def test_ortho_error_closed_form():
    assert oracle.ortho_error(np.eye(5)[:, :3]) == 0.0
    assert abs(oracle.ortho_error(arr([[1.0, 1.0], [0.0, 0.0]])) - 1.0) <= 1e-15


# ------------------------------------------------- SPEC tssvd closed forms --
@pytest.mark.parametrize("passes", [1, 2])
def test_tssvd_spec_examples(passes):
    e = SPEC["ts_svd_gram_diag"]
    u, s, v = oracle.tssvd(arr(e["A"]), passes=passes)
    assert np.max(np.abs(s - arr(e["sigma"]))) <= 1e-15
    e = SPEC["ts_svd_gram_double_identity"]
    a = arr(e["A"])
    u, s, v = oracle.tssvd(a, passes=passes)
    assert oracle.ortho_error(u) <= e["ortho_max"]
    assert np.max(np.abs(np.abs(u @ v.T) - a)) <= 1e-14  # U V^T reproduces the input


# ---------------------------------------------------- constructed spectra --
@pytest.mark.parametrize("wp,r", [(1e-11, 9), (1e-14, 10)])
def test_c1_constructed_spectrum(wp, r):
    """c1: sigma_j = 10^(-6(j-1)/9); sigma_10 = 1e-6 < sqrt(1e-11) drops, kept at wp=1e-14."""
    d = synth.config_inputs("c1")
    a, s = d["A"], d["sigma"]
    v_true = synth.haar(10, 10, 1, synth.matrices.STREAM_V)
    u_true = synth.haar(4000, 10, 1, synth.matrices.STREAM_U)
    u3, s3, v3 = oracle.tssvd(a, wp, passes=1)
    u4, s4, v4 = oracle.tssvd(a, wp, passes=2)
    for uu, ss, vv in ((u3, s3, v3), (u4, s4, v4)):
        assert ss.size == r
        assert np.max(np.abs(ss - s[:r])) <= 1e-12 * s[0]
        assert np.all(np.diff(ss) < 0)
        assert oracle.ortho_error(vv) <= 1e-13
        for j in range(r):  # sign-invariant column comparison, bound of reading Q11
            bound = 1e3 * EPS * (s[0] / s[j]) ** 2
            assert min(np.linalg.norm(vv[:, j] - v_true[:, j]), np.linalg.norm(vv[:, j] + v_true[:, j])) <= bound
            assert min(np.linalg.norm(uu[:, j] - u_true[:, j]), np.linalg.norm(uu[:, j] + u_true[:, j])) <= bound
    # explicit normalisation (Remark 'normalizing'): unit columns to ~eps even after 1 pass
    assert np.max(np.abs(np.sum(u3 * u3, axis=0) - 1.0)) <= 1e-14
    # one pass loses orthonormality (off-diagonal ~1e-7), the second pass restores it (Tables 3-5)
    assert oracle.ortho_error(u3) >= 1e-9
    assert oracle.ortho_error(u4) <= 1e-13
    # reconstruction: ||A - U S V^T||_2 = sigma_{r+1} (or ~eps when nothing is dropped)
    res = np.linalg.norm(a - (u4 * s4) @ v4.T, 2)
    expect = s[r] if r < 10 else 0.0
    assert abs(res - expect) <= 1e-3 * s[min(r, 9)]


def test_c2_reduced_constructed_spectrum():
    """c2 recipe at m = 2e5: r = 55 (sigma_55 = 3.51e-6 > 3.16e-6 > sigma_56 = 2.78e-6)."""
    d = synth.config_inputs("c2", m=200_000)
    a, s = d["A"], d["sigma"]
    u, sg, v = oracle.tssvd(a, 1e-11, passes=2)
    assert sg.size == 55
    assert np.max(np.abs(sg - s[:55])) <= 1e-12
    assert oracle.ortho_error(u) <= 1e-13
    assert oracle.ortho_error(v) <= 1e-13
    _, _, _, y = oracle.alg4(a, 1e-11, return_pass1=True)
    assert 1e-9 <= oracle.ortho_error(y) <= 1e-4  # pass 1 ~ half the digits


@pytest.mark.parametrize("parts", [2, 4, 8])
def test_shard_invariance(parts):
    """Partition count changes only rounding (SPEC.md:538 analogue)."""
    d = synth.config_inputs("c2", m=40_000)
    a = d["A"]
    u1, s1, v1 = oracle.tssvd(a, 1e-11, 2, parts=1)
    up, sp, vp = oracle.tssvd(a, 1e-11, 2, parts=parts)
    assert sp.size == s1.size
    assert np.max(np.abs(sp - s1)) <= 1e-14
    assert oracle.ortho_error(up, parts) <= 1e-13


def test_brute_force_tiny_random_vs_lapack_svd():
    """50 random inputs <= 200 x 30 incl. rank-deficient, duplicate columns and zero."""
    rng = np.random.default_rng(5)
    for case in range(50):
        m = int(rng.integers(30, 201))
        n = int(rng.integers(1, 31))
        a = rng.standard_normal((m, n))
        if case % 5 == 1 and n > 2:
            a[:, : n // 2] = a[:, : n // 2] @ np.diag(10.0 ** -rng.uniform(0, 12, n // 2))
        if case % 5 == 2 and n > 3:
            a = a[:, :3] @ rng.standard_normal((3, n))  # rank 3
        if case % 5 == 3 and n > 1:
            a[:, -1] = a[:, 0]  # duplicate column
        if case == 4:
            a[:] = 0.0
        wp = 1e-11
        s_true = np.linalg.svd(a, compute_uv=False)
        u, s, v = oracle.tssvd(a, wp, passes=2)
        assert np.all(np.isfinite(u)) and np.all(np.isfinite(s)) and np.all(np.isfinite(v))
        if s_true[0] == 0.0:
            assert s.size == 0
            continue
        big = s_true >= 1e-3 * s_true[0]  # clear of the sqrt(wp) threshold
        assert s.size >= big.sum()
        assert np.max(np.abs(s[: big.sum()] - s_true[big])) <= 1e-8 * s_true[0]
        assert oracle.ortho_error(u) <= 1e-13 and oracle.ortho_error(v) <= 1e-13
        assert np.linalg.norm(a - (u * s) @ v.T, 2) <= 1e-5 * s_true[0]


def test_argument_errors():
    with pytest.raises(ValueError):
        oracle.tssvd(np.ones((2, 3)))  # wide
    with pytest.raises(ValueError):
        oracle.tssvd(arr([[np.nan], [1.0]]))
    with pytest.raises(ValueError):
        oracle.tssvd(np.ones((3, 1)), wp=0.0)
    with pytest.raises(ValueError):
        oracle.lowrank_svd(np.ones((5, 4)), np.ones((4, 4)), 1)  # l >= min(m, n)


def test_canonical_signs():
    rng = np.random.default_rng(6)
    u = rng.standard_normal((7, 3))
    v = rng.standard_normal((4, 3))
    cu, cv = oracle.canonical_signs(u, v)
    for j in range(3):
        i = np.argmax(np.abs(cv[:, j]))
        assert cv[i, j] > 0
        assert np.array_equal(cu[:, j] * cv[0, j], u[:, j] * v[0, j])


# ------------------------------------------------------------ low rank ----
def test_lowrank_c3_reduced_known_spectrum():
    """c3 recipe at 2e4 x 4e3: leading sigma and err_k = sigma_{k+1} = 1e-2 (no discards)."""
    d = synth.config_inputs("c3", m=20_000, n=4_000)
    u, s, v = oracle.lowrank_svd(d["A"], d["Omega"], d["iters"], d["k"])
    assert s.size == d["k"]
    assert np.max(np.abs(s - d["sigma"][: d["k"]])) <= 1e-6  # noise level 1e-6
    err = oracle.spectral_error(d["A"], u, s, v, d["x0"])
    assert abs(err - d["sigma"][d["k"]]) <= 1e-3 * d["sigma"][d["k"]]
    assert oracle.ortho_error(u) <= 1e-13 and oracle.ortho_error(v) <= 1e-13


def test_lowrank_i0_and_exact_rank_capture():
    """i = 0 skips the loop (reading Q7); an exactly rank-3 A is captured to ~eps."""
    rng = np.random.default_rng(7)
    a = rng.standard_normal((300, 3)) @ rng.standard_normal((3, 80))
    om = rng.standard_normal((80, 6))
    for i in (0, 1, 2):
        u, s, v = oracle.lowrank_svd(a, om, i, 6)
        assert s.size == 3  # the three noise directions are discarded by the sqrt(wp) rule
        assert np.linalg.norm(a - (u * s) @ v.T, 2) <= 1e-9 * s[0]


@pytest.mark.slow
def test_paper_table8_alg8_l20():
    """Algorithm 8, m=1e4, n=2000, l=20, i=2 -> ||A-USV*|| = 4.83e-07 (= sigma_7)."""
    g = PAPER["alg8_l20_i2_m1e4_n2000"]
    a, sig = synth.paper_lowrank_test_matrix(g["m"], g["n"], g["l"])
    om = synth.omega(g["n"], g["l"], 100)  # recorded seed: kept rank 6 (reading P5)
    u, s, v = oracle.lowrank_svd(a, om, g["i"], g["l"])
    err = oracle.spectral_error(a, u, s, v, synth.power_start(g["n"], 7))
    assert s.size == 6
    assert round(err, 9) == pytest.approx(g["spectral_error"], rel=5e-3)
    assert abs(err - sig[6]) <= 1e-3 * sig[6]
    assert oracle.ortho_error(u) <= 1e-13 and oracle.ortho_error(v) <= 1e-13


@pytest.mark.slow
def test_paper_table10_alg8_l10():
    """Algorithm 8 with l=10, i=2 -> 2.15e-07 (= sigma_4 of Eq. testSl)."""
    g = PAPER["alg8_l10_i2"]
    a, sig = synth.paper_lowrank_test_matrix(10_000, 2_000, g["l"])
    for seed in (100, 101):
        u, s, v = oracle.lowrank_svd(a, synth.omega(2_000, g["l"], seed), g["i"], g["l"])
        err = oracle.spectral_error(a, u, s, v, synth.power_start(2_000, 7))
        assert s.size == 3
        assert err == pytest.approx(g["spectral_error"], rel=5e-3)


@pytest.mark.slow
def test_paper_table5_alg4():
    """Algorithm 4, m=1e4, n=2000 -> error ~9.64e-07, max|U*U-I| ~6.66e-15.

    Orders of magnitude only (the paper's wp for this table is ~1e-12, reading Q1).
    """
    g = PAPER["alg4_m1e4_n2000"]
    a, sig = synth.paper_test_matrix(g["m"], g["n"])
    u, s, v = oracle.tssvd(a, 1e-12, passes=2)
    err = oracle.spectral_error(a, u, s, v, synth.power_start(g["n"], 7))
    assert err == pytest.approx(g["spectral_error"], rel=0.05)
    assert oracle.ortho_error(u) <= 10 * g["max_UtU_minus_I"]
    assert oracle.ortho_error(v) <= 10 * g["max_VtV_minus_I"]


def test_devils_staircase_recipe():
    """PAPER.md:1351-1368 (the Scala recipe): every value is a multiple of 1/63 in [0, 1], the
    binary image of the octal digits (1-7 -> 1) of round(j 8^6 / k); j = 0 is the only zero for
    k = 2000; small k by hand: k = 8 -> round(j 8^5) octal j00000 -> binary j>0 ? 100000 : 0."""
    g = PAPER["staircase_values"]
    s = synth.devils_staircase(2000)
    b = s * g["denominator"]
    assert np.allclose(b, np.round(b), atol=1e-12) and s.max() == g["max"] and s.min() == 0.0
    assert int(np.sum(s == 0.0)) == g["zeros_for_k_2000"]
    assert np.all(np.diff(s) <= 0)
    k8 = synth.devils_staircase(8)
    assert np.allclose(k8, [32 / 63] * 7 + [0.0])


@pytest.mark.slow
@pytest.mark.parametrize("passes,key", [(1, "staircase_alg3_m1e4_n2000"), (2, "staircase_alg4_m1e4_n2000")])
def test_paper_table21_staircase(passes, key):
    """PAPER.md:1457-1458 (Table 21, Devil's staircase, m = 1e4, n = 2000): residual ~1e-14 and
    orthonormality at the printed orders of magnitude; the kept rank drops only the one zero."""
    g = PAPER[key]
    a, sig = synth.paper_staircase_matrix(g["m"], g["n"])
    u, s, v = oracle.tssvd(a, 1e-11, passes)
    err = oracle.spectral_error(a, u, s, v, synth.power_start(g["n"], 7))
    assert s.size == g["n"] - 1
    assert g["spectral_error"] / 10 <= err <= 10 * g["spectral_error"]
    assert oracle.ortho_error(u) <= 10 * g["max_UtU_minus_I"]
    assert oracle.ortho_error(v) <= 10 * g["max_VtV_minus_I"]
    assert np.max(np.abs(s - sig[: s.size])) <= 1e-12


# ------------------------------------------ Algorithms 1, 2, 7 (TSQR) --
def test_mixing_closed_forms():
    """Remark 'randomness': Omega = D F S D~ F S~ on pairs viewed as complex numbers.
    n = 2 (h = 1: F = 1, S = id): a plane rotation by theta_D + theta_D~; n = 4 (h = 2:
    F = [[1, 1], [1, -1]] / sqrt 2) written out by hand; any n: orthogonal, norm-preserving, and
    the inverse map undoes it; odd n leaves the last entry alone (reading R17)."""
    ph = np.array([0.3, 1.1])
    om = oracle.mix_rows(np.eye(2), ph, np.array([0, 0]))
    c, s = np.cos(1.4), np.sin(1.4)
    assert np.allclose(om, [[c, s], [-s, c]], atol=1e-15)  # row k = Omega e_k
    ph = np.array([0.2, 0.7, 1.3, 2.9])
    pm = np.array([1, 0, 0, 1])  # S swaps, S~ = id
    x = np.array([0.5, -1.0, 2.0, 0.25])
    z = np.array([x[0] + 1j * x[1], x[2] + 1j * x[3]])
    f = np.array([[1, 1], [1, -1]]) / np.sqrt(2)
    z = f @ z                                  # F S~ z (S~ = id)
    z = np.exp(1j * ph[2:]) * z                # D~
    z = z[[1, 0]]                              # S
    z = np.exp(1j * ph[:2]) * (f @ z)          # D F
    want = np.array([z[0].real, z[0].imag, z[1].real, z[1].imag])
    assert np.allclose(oracle.mix_rows(x[None, :], ph, pm)[0], want, atol=1e-15)
    for n in (10, 37, 100):
        ph, pm = synth.mixing_params(n, 3)
        om = oracle.mix_rows(np.eye(n), ph, pm)
        assert np.max(np.abs(om @ om.T - np.eye(n))) <= 1e-14
        assert np.max(np.abs(oracle.mix_rows(om, ph, pm, inverse=True) - np.eye(n))) <= 1e-14
        if n % 2:
            assert om[n - 1, n - 1] == 1.0 and np.all(om[n - 1, :n - 1] == 0.0)
        for half in range(2):
            assert sorted(pm[half * (n // 2):(half + 1) * (n // 2)]) == list(range(n // 2))


@pytest.mark.parametrize("alg", ["alg1", "alg2"])
def test_alg12_constructed_and_tiny(alg):
    """Alg. 1 / 2 on c1's constructed spectrum (sigma, U, V against the true
    factors: QR-based, so no squaring of the condition number -- sigma to 1e-15 sigma_1) and on
    random tiny matrices against numpy's SVD of A itself."""
    f = getattr(oracle, alg)
    d = synth.config_inputs("c1")
    ph, pm = synth.mixing_params(10, 1)
    u, s, v = f(d["A"], ph, pm, 1e-11)
    assert s.size == 10
    assert np.max(np.abs(s - d["sigma"])) <= 1e-15 * 4
    assert oracle.ortho_error(u) <= 1e-14 and oracle.ortho_error(v) <= 1e-14
    assert np.max(np.abs(d["A"] - (u * s) @ v.T)) <= 1e-15 * 10
    rng = np.random.default_rng(7)
    for trial in range(20):
        m, n = int(rng.integers(5, 60)), int(rng.integers(1, 5)) * 2
        m = max(m, n)
        a = rng.standard_normal((m, n))
        ph, pm = synth.mixing_params(n, trial)
        u, s, v = f(a, ph, pm, 1e-11)
        ref = np.linalg.svd(a, compute_uv=False)
        assert np.allclose(s, ref, rtol=1e-12, atol=1e-13 * ref[0])
        assert np.max(np.abs(a - (u * s) @ v.T)) <= 1e-13 * ref[0]


@pytest.mark.slow
@pytest.mark.parametrize("alg,key", [("alg1", "alg1_m1e4_n2000"), ("alg2", "alg2_m1e4_n2000")])
def test_paper_table5_alg12(alg, key):
    """PAPER.md:970-971 (Table 5, Algorithms 1 and 2, m = 1e4, n = 2000): residual 9.76e-12.  The
    kept rank follows R's diagonal against R_11 wp, which depends on the random Omega, so the
    residual (~ the first dropped sigma, ~1e-11) is pinned to 10%; V orthonormality to 10x."""
    g = PAPER[key]
    a, sig = synth.paper_test_matrix(g["m"], g["n"])
    u, s, v = getattr(oracle, alg)(a, *synth.mixing_params(g["n"], 1), 1e-11)
    err = oracle.spectral_error(a, u, s, v, synth.power_start(g["n"], 7))
    assert err == pytest.approx(g["spectral_error"], rel=0.1)
    assert oracle.ortho_error(v) <= 10 * g["max_VtV_minus_I"]


@pytest.mark.slow
@pytest.mark.parametrize("key,l", [("alg7_l20_i2_m1e4_n2000", 20), ("alg7_l10_i2", 10)])
def test_paper_alg7(key, l):
    """PAPER.md:1039 and 1084-1087 (Tables 8 and 10, Algorithm 7): the residual is exactly
    sigma_{r+1} of Eq. testSl -- 2.64e-12 = sigma_12 (l = 20) and 7.74e-12 = sigma_6 (l = 10) --
    with the recorded seeds that give the paper's kept ranks (11 and 5)."""
    g = PAPER[key]
    a, sig = synth.paper_lowrank_test_matrix(10_000, 2_000, l)
    seed = g["seed"]
    u, s, v = oracle.lowrank_svd_tsqr(a, synth.omega(2_000, l, seed), g["i"], l,
                                      lambda w: synth.mixing_params(w, seed), 1e-11)
    err = oracle.spectral_error(a, u, s, v, synth.power_start(2_000, 7))
    assert err == pytest.approx(g["spectral_error"], rel=5e-3)
    assert abs(err - sig[s.size]) <= 1e-3 * sig[s.size]
    assert oracle.ortho_error(u) <= 1e-14 and oracle.ortho_error(v) <= 1e-14


# ----------------------------------------------- LU-based subspace tracking --
def test_lu_tracking_factor_is_lapack_gepp():
    """P:405-409 (reading R21): the L of Gaussian elimination with partial pivoting.  Special
    case that reduces to a library routine: LAPACK dgetrf (scipy.linalg.lu, Y = P L U) picks the
    same pivots, so the oracle's L (Y's row order) equals P L; partial pivoting bounds |L| <= 1;
    the column space of L is Y's (projection residual at rounding level)."""
    import scipy.linalg as sl

    rng = np.random.default_rng(21)
    for m, l in [(50, 6), (400, 25), (1000, 60), (7, 7)]:
        y = rng.standard_normal((m, l)) * np.logspace(0, -4, l)[None, :]
        lm, r = oracle.lu_tracking_factor(y, 1e-11)
        p, ls, u = sl.lu(y)
        assert r == l
        assert np.max(np.abs(lm - p @ ls)) <= 1e-13
        assert np.max(np.abs(lm)) <= 1.0
        q = np.linalg.qr(lm)[0]
        assert np.linalg.norm(y - q @ (q.T @ y), 2) <= 1e-13 * np.linalg.norm(y, 2)


def test_lu_tracking_factor_rank_deficient():
    """A numerically zero pivot stops the elimination (R21): rank-3 Y with 6 columns keeps 3
    columns spanning Y's column space; Y = 0 keeps none."""
    rng = np.random.default_rng(22)
    y = rng.standard_normal((300, 3)) @ rng.standard_normal((3, 6))
    lm, r = oracle.lu_tracking_factor(y, 1e-11)
    assert r == 3 and lm.shape == (300, 3)
    q = np.linalg.qr(lm)[0]
    assert np.linalg.norm(y - q @ (q.T @ y), 2) <= 1e-12 * np.linalg.norm(y, 2)
    assert oracle.lu_tracking_factor(np.zeros((10, 4)))[1] == 0


def test_lowrank_lu_equals_alg8():
    """'the column space of L is the same as the column space of Q', so Alg. 8 with
    LU tracking returns Alg. 8's result: on c3's spectrum (reduced; no singular value near the
    sqrt(wp) discard line) sigma agrees to 1e-13 sigma_1 and U, V columns within the R12 bound.
    (Near the line the variant can differ: on the paper's Table 8 matrix sigma_6 / sigma_1 = 5.5e-6
    is 1.7x above it and the LU variant keeps 5 where Alg. 8 keeps 6 -- DESIGN.md R21.)"""
    d = synth.config_inputs("c3", m=20_000, n=2_000)
    ref = oracle.lowrank_svd(d["A"], d["Omega"], d["iters"], d["k"])
    lu = oracle.lowrank_svd_lu(d["A"], d["Omega"], d["iters"], d["k"])
    assert lu[1].size == ref[1].size
    assert np.max(np.abs(lu[1] - ref[1])) <= 1e-13 * ref[1][0]
    bound = 1e3 * np.finfo(float).eps * (ref[1][0] / ref[1]) ** 2
    for g, r in ((lu[0], ref[0]), (lu[2], ref[2])):
        dist = np.minimum(np.linalg.norm(g - r, axis=0), np.linalg.norm(g + r, axis=0))
        assert np.all(dist <= bound)
