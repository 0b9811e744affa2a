"""Pins of the CPU oracle against what the paper and the mathematics fix.

The paper prints no coefficient values, so the oracle is pinned by
(P1) brute force from the operator definitions, (P2) the separable special case
computed by a textbook fold+FFT algorithm, (P3) the delta-window closed form,
(P4) single-atom inputs, (P5/P6) modulation / translation covariance, (P7) real
input symmetry, (P8) the energy identity for the canonical tight window and (P9)
perfect reconstruction with the canonical dual (dense linear algebra, PAPER.md:
167-176).  Each pin is chosen so a dropped term, a wrong sign, a wrong index or a
transposed operand fails at least one of them.
"""
import math

import numpy as np
import pytest

import dense
from synthetic import pgauss, random_pair

# Fig. 1 lattices: a=6, M=6, L=36, lambda in {0, 1/2, 1/3, 2/3}.
FIG1 = [(36, 6, 6, 0, 1), (36, 6, 6, 1, 2), (36, 6, 6, 1, 3), (36, 6, 6, 2, 3)]
TINY = FIG1 + [
    (24, 4, 6, 1, 2), (48, 6, 8, 1, 2), (60, 10, 15, 1, 2), (72, 8, 12, 1, 3),
    (108, 9, 12, 2, 3), (48, 4, 12, 1, 4), (100, 4, 10, 1, 5), (64, 8, 16, 3, 4),
    (240, 8, 12, 1, 2),  # config 1 shape
]


def rel(x, y):
    return float(np.linalg.norm(x - y) / np.linalg.norm(y))


@pytest.mark.parametrize("L,a,M,l1,l2", TINY)
@pytest.mark.parametrize("variant", ["literal", "regrouped"])
def test_dense_atoms(oracle_mod, L, a, M, l1, l2, variant):
    """P1: c = G^H f with atoms M_{sn+bk} T_{an} g built from PAPER.md:151-158, 195."""
    f, g = random_pair(L, 11)
    c = oracle_mod.dgt(f, g, a, M, l1, l2, variant=variant)
    ref = dense.dense_dgt(f, g, a, M, l1, l2)
    assert rel(c, ref) < 1e-12


@pytest.mark.parametrize("L,a,M", [(24, 4, 6), (120, 10, 12), (240, 8, 12), (480, 16, 24), (1024, 32, 64)])
def test_separable_textbook(oracle_mod, L, a, M):
    """P2: lambda=[0,1] equals the textbook separable DGT c(.,n) = FFT_M(fold_M(f conj(T_an g)))."""
    f, g = random_pair(L, 12)
    c = oracle_mod.dgt(f, g, a, M, 0, 1)
    N = L // a
    ref = np.zeros((M, N), complex)
    l = np.arange(L)
    for n in range(N):
        h = f.astype(complex) * np.conj(g[(l - a * n) % L])
        ref[:, n] = np.fft.fft(h.reshape(L // M, M).sum(axis=0))
    assert rel(c, ref) < 1e-12


def _w(n, l1, l2):
    return ((n * l1) % l2) / l2


@pytest.mark.parametrize("L,a,M,l1,l2", [(36, 6, 6, 1, 3), (240, 8, 12, 1, 2), (2880, 60, 240, 1, 3),
                                         (14400, 50, 200, 1, 2)])
def test_delta_window(oracle_mod, L, a, M, l1, l2):
    """P3: g = delta_0  =>  c(m,n) = f(an) exp(-2 pi i (m + w(n)) a n / M)."""
    f, _ = random_pair(L, 13)
    g = np.zeros(L, complex)
    g[0] = 1.0
    N = L // a
    cols = np.arange(0, N, max(1, N // 37))
    c = oracle_mod.dgt(f, g, a, M, l1, l2, cols=cols)
    m = np.arange(M)[:, None]
    n = cols[None, :]
    w = ((n * l1) % l2) / l2
    ref = f[a * n] * np.exp(-2j * np.pi * ((m + w) * a * n % M) / M)
    assert rel(c, ref) < 1e-12


@pytest.mark.parametrize("L,a,M,l1,l2", [(36, 6, 6, 1, 2), (72, 8, 12, 1, 3), (240, 8, 12, 1, 2)])
def test_single_atom(oracle_mod, L, a, M, l1, l2):
    """P4: f = M_{b(m0+w(n0))} T_{a n0} g  =>  c(m0, n0) = ||g||^2."""
    _, g = random_pair(L, 14)
    b = L // M
    N = L // a
    rng = np.random.default_rng(5)
    for _ in range(5):
        m0, n0 = int(rng.integers(M)), int(rng.integers(N))
        s = b * l1 // l2
        om = (b * m0 + (s * n0) % b)
        f = dense.atom(g, a * n0, om)
        c = oracle_mod.dgt(f, g, a, M, l1, l2)
        assert abs(c[m0, n0] - np.vdot(g, g)) < 1e-12


@pytest.mark.parametrize("L,a,M,l1,l2", [(72, 8, 12, 1, 3), (240, 8, 12, 1, 2), (1440, 30, 48, 2, 3)])
def test_modulation_covariance(oracle_mod, L, a, M, l1, l2):
    """P5: f' = exp(2 pi i l / M) f  =>  c'(m, n) = c(m-1 mod M, n)."""
    f, g = random_pair(L, 15)
    l = np.arange(L)
    c = oracle_mod.dgt(f, g, a, M, l1, l2)
    c2 = oracle_mod.dgt(np.exp(2j * np.pi * l / M) * f, g, a, M, l1, l2)
    assert rel(c2, np.roll(c, 1, axis=0)) < 1e-12


@pytest.mark.parametrize("L,a,M,l1,l2", [(72, 8, 12, 1, 3), (240, 8, 12, 1, 2), (1440, 30, 48, 2, 3)])
def test_translation_covariance(oracle_mod, L, a, M, l1, l2):
    """P6: f' = f(. - lambda2 a)  =>  c'(m,n) = exp(-2 pi i (m+w(n)) lambda2 a / M) c(m, n - lambda2)."""
    f, g = random_pair(L, 16)
    c = oracle_mod.dgt(f, g, a, M, l1, l2)
    c2 = oracle_mod.dgt(np.roll(f, l2 * a), g, a, M, l1, l2)
    N = L // a
    m = np.arange(M)[:, None]
    n = np.arange(N)[None, :]
    w = ((n * l1) % l2) / l2
    ref = np.exp(-2j * np.pi * (m + w) * l2 * a / M) * np.roll(c, l2, axis=1)
    assert rel(c2, ref) < 1e-12


@pytest.mark.parametrize("L,a,M,l1,l2", [(240, 8, 12, 1, 2), (96, 8, 12, 0, 1), (480, 16, 24, 1, 2)])
def test_real_input_symmetry(oracle_mod, L, a, M, l1, l2):
    """P7: real f, real g, lambda2 <= 2  =>  conj(c(m,n)) = c((-m - 2 w(n)) mod M, n)."""
    rng = np.random.default_rng(17)
    f = rng.standard_normal(L)
    g = pgauss(L, a * M / L)
    c = oracle_mod.dgt(f, g, a, M, l1, l2)
    N = L // a
    for n in range(N):
        two_w = (2 * ((n * l1) % l2)) // l2
        idx = (-np.arange(M) - two_w) % M
        assert np.allclose(np.conj(c[:, n]), c[idx, n], atol=1e-12 * np.abs(c).max())


@pytest.mark.parametrize("L,a,M,l1,l2", [(48, 6, 12, 1, 2), (72, 8, 12, 1, 3), (240, 8, 12, 1, 2),
                                         (120, 10, 20, 1, 2)])
def test_energy_tight(oracle_mod, L, a, M, l1, l2):
    """P8: for the canonical tight window g_t = S^{-1/2} g, ||c||^2 = ||f||^2, and for
    any scaling t*g_t: ||c||^2 = (M N / L) ||t g_t||^2 ||f||^2."""
    g = pgauss(L, a * M / L)
    gt = oracle_mod.windows.canonical_tight(g, a, M, l1, l2)
    f, _ = random_pair(L, 18)
    c = oracle_mod.dgt(f, gt, a, M, l1, l2)
    assert abs(np.vdot(c, c).real - np.vdot(f, f).real) < 1e-11 * np.vdot(f, f).real
    N = L // a
    assert abs(M * N / L * np.vdot(gt, gt).real - 1.0) < 1e-11
    t = 0.37
    c2 = oracle_mod.dgt(f, t * gt, a, M, l1, l2)
    assert abs(np.vdot(c2, c2).real - M * N / L * t * t * np.vdot(gt, gt).real * np.vdot(f, f).real) \
        < 1e-11 * np.vdot(f, f).real


@pytest.mark.parametrize("L,a,M,l1,l2", [(36, 6, 6, 1, 2), (36, 6, 12, 1, 3), (72, 8, 12, 1, 3),
                                         (240, 8, 12, 1, 2)])
def test_perfect_reconstruction(oracle_mod, L, a, M, l1, l2):
    """P9: f = sum c(m,n) M_{b(m+w(n))} T_{an} gamma with gamma = S^{-1} g.
    Includes config 1 itself (L=240, a=8, M=12, quincunx, pgauss with tfr = aM/L)."""
    g = pgauss(L, a * M / L)
    gamma = oracle_mod.windows.canonical_dual(g, a, M, l1, l2)
    f, _ = random_pair(L, 19)
    c = oracle_mod.dgt(f, g, a, M, l1, l2)
    f_rec = dense.synthesize(c, gamma, a, M, l1, l2)
    assert rel(f_rec, f.astype(complex)) < 1e-11


@pytest.mark.parametrize("L,a,M,l1,l2", [(36, 6, 6, 1, 2), (216, 12, 18, 1, 3), (400, 50, 200, 1, 2),
                                         (720, 60, 240, 1, 3), (512, 64, 256, 1, 2)])
def test_literal_equals_regrouped(oracle_mod, L, a, M, l1, l2):
    """O1 (literal) and O2 (regrouped) evaluate the same finite sum."""
    f, g = random_pair(L, 20)
    c1 = oracle_mod.dgt(f, g, a, M, l1, l2, variant="literal")
    c2 = oracle_mod.dgt(f, g, a, M, l1, l2, variant="regrouped")
    assert rel(c1, c2) < 1e-13


def test_column_subset_and_batch(oracle_mod):
    """Sampled columns and batched signals equal the full single-signal result."""
    L, a, M, l1, l2 = 720, 60, 240, 1, 3
    f1, g = random_pair(L, 21)
    f2, _ = random_pair(L, 22)
    full = oracle_mod.dgt(np.stack([f1, f2]), g, a, M, l1, l2)
    cols = [0, 5, 11]
    sub = oracle_mod.dgt(np.stack([f1, f2]), g, a, M, l1, l2, cols=cols)
    assert np.array_equal(sub, full[:, :, cols])
    assert np.array_equal(full[1], oracle_mod.dgt(f2, g, a, M, l1, l2))


def test_rejects_infeasible(oracle_mod):
    f, g = random_pair(36, 1)
    with pytest.raises(ValueError):
        oracle_mod.dgt(f, g, 6, 6, 1, 4)   # lambda2=4 does not divide b=6
    with pytest.raises(ValueError):
        oracle_mod.dgt(f, g, 5, 6, 0, 1)   # a does not divide L


def test_config1_window_properties():
    """The config-1 window (Z14): real, even, unit norm."""
    g = pgauss(240, 8 * 12 / 240)
    assert abs(np.linalg.norm(g) - 1) < 1e-14
    assert np.allclose(g[1:], g[1:][::-1], rtol=0, atol=1e-15)
    assert math.isclose(g[0], g.max())


# ---- synthesis (inverse DGT): oracle.idgt ----

@pytest.mark.parametrize("L,a,M,l1,l2", TINY)
@pytest.mark.parametrize("variant", ["literal", "regrouped"])
def test_idgt_dense_atoms(oracle_mod, L, a, M, l1, l2, variant):
    """S1/S2 against the dense synthesis matrix whose columns are the atoms
    M_{sn+bk} T_{an} gamma built from the operator definitions."""
    rng = np.random.default_rng(L + 7 * M + l1)
    N = L // a
    c = rng.standard_normal((M, N)) + 1j * rng.standard_normal((M, N))
    _, gamma = random_pair(L, 31)
    ref = dense.synthesize(c, gamma, a, M, l1, l2)
    assert rel(oracle_mod.idgt(c, gamma, a, M, l1, l2, variant=variant), ref) < 1e-12


@pytest.mark.parametrize("L,a,M,l1,l2", [(72, 8, 12, 1, 3), (240, 8, 12, 1, 2), (1440, 30, 48, 2, 3),
                                         (2880, 60, 240, 1, 3)])
def test_idgt_is_adjoint_of_dgt(oracle_mod, L, a, M, l1, l2):
    """<dgt(f, g), c> = <f, idgt(c, g)> for random f, c (the synthesis operator is the adjoint
    of the analysis operator with the same window; dgt is pinned independently above)."""
    rng = np.random.default_rng(L)
    f, g = random_pair(L, 33)
    N = L // a
    c = rng.standard_normal((M, N)) + 1j * rng.standard_normal((M, N))
    lhs = np.vdot(c, oracle_mod.dgt(f, g, a, M, l1, l2))          # <dgt f, c> conj-linear in c
    rhs = np.vdot(oracle_mod.idgt(c, g, a, M, l1, l2), f)         # <f, idgt c>
    assert abs(lhs - rhs) <= 1e-11 * abs(lhs)


@pytest.mark.parametrize("L,a,M,l1,l2", [(36, 6, 6, 1, 2), (72, 8, 12, 1, 3), (240, 8, 12, 1, 2)])
def test_idgt_perfect_reconstruction(oracle_mod, L, a, M, l1, l2):
    """idgt(dgt(f, g), S^{-1} g) = f (inversion formula), the dual from the
    dense frame operator."""
    g = pgauss(L, a * M / L)
    gamma = oracle_mod.windows.canonical_dual(g, a, M, l1, l2)
    f, _ = random_pair(L, 34)
    f_rec = oracle_mod.idgt(oracle_mod.dgt(f, g, a, M, l1, l2), gamma, a, M, l1, l2)
    assert rel(f_rec, f.astype(complex)) < 1e-11


@pytest.mark.parametrize("L,a,M,l1,l2", [(216, 12, 18, 1, 3), (720, 60, 240, 1, 3), (512, 64, 256, 1, 2)])
def test_idgt_literal_equals_regrouped_batch(oracle_mod, L, a, M, l1, l2):
    rng = np.random.default_rng(5)
    N = L // a
    c = rng.standard_normal((2, M, N)) + 1j * rng.standard_normal((2, M, N))
    _, gamma = random_pair(L, 35)
    f1 = oracle_mod.idgt(c, gamma, a, M, l1, l2, variant="literal")
    f2 = oracle_mod.idgt(c, gamma, a, M, l1, l2, variant="regrouped")
    assert f1.shape == (2, L) and rel(f1, f2) < 1e-13
    assert rel(oracle_mod.idgt(c[1], gamma, a, M, l1, l2), f2[1]) < 1e-13


# ---- canonical dual / tight windows: oracle.windows ----

# redundancy M/a > 1 (the Fig. 1 lattices are critically sampled; there the Gaussian system is
# a near-singular frame and reconstruction is ill-conditioned)
@pytest.mark.parametrize("L,a,M,l1,l2", [(36, 6, 12, 1, 3), (36, 4, 6, 1, 3), (36, 6, 12, 2, 3), (72, 8, 12, 1, 3),
                                         (240, 8, 12, 1, 2), (120, 10, 12, 0, 1), (96, 8, 12, 1, 4)])
def test_dual_window_defining_equation(oracle_mod, L, a, M, l1, l2):
    """S gamma = g with S applied as idgt(dgt(., g), g) (the oracle's own, independently pinned
    analysis and synthesis sums), and perfect reconstruction with gamma."""
    g = pgauss(L, a * M / L)
    gamma = oracle_mod.windows.canonical_dual(g, a, M, l1, l2)
    Sg = oracle_mod.idgt(oracle_mod.dgt(gamma, g, a, M, l1, l2), g, a, M, l1, l2)
    assert rel(Sg, g.astype(complex)) < 1e-11
    f, _ = random_pair(L, 36)
    fr = oracle_mod.idgt(oracle_mod.dgt(f, g, a, M, l1, l2), gamma, a, M, l1, l2)
    assert rel(fr, f.astype(complex)) < 1e-11


@pytest.mark.parametrize("L,a,M,l1,l2", [(36, 6, 6, 1, 2), (72, 8, 12, 1, 3), (240, 8, 12, 1, 2)])
def test_tight_window_properties(oracle_mod, L, a, M, l1, l2):
    """g_t = S^{-1/2} g: the system of g_t is a Parseval frame -- perfect reconstruction with
    itself and ||c||^2 = ||f||^2 (S_{g_t} = I)."""
    g = pgauss(L, a * M / L)
    gt = oracle_mod.windows.canonical_tight(g, a, M, l1, l2)
    f, _ = random_pair(L, 37)
    c = oracle_mod.dgt(f, gt, a, M, l1, l2)
    assert abs(np.linalg.norm(c) ** 2 / np.linalg.norm(f) ** 2 - 1.0) < 1e-11
    assert rel(oracle_mod.idgt(c, gt, a, M, l1, l2), f.astype(complex)) < 1e-11
