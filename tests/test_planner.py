"""Host planner (C ABI ``dgt_lattice_plan``): feasibility, shear validity, constants.

Pins: the printed remark numbers (tests/golden/paper_remark_examples.txt, PAPER.md:
721-734), brute force over L for Prop. minsig, brute force over
(s0, s1) in Z_L^2 for the existence of a time-only shear, and the lattice identity
U^{-1}_{s0,s1} A Z_L^2 = D Z_L^2 with D = diag(ab/X, X) (Thm. shearform and its proof,
PAPER.md:457-531) checked as point sets -- independent of Algorithm 1.
"""
import math
import os

import pytest

import paper_1307_4569_b200 as nsdgt
from paper_1307_4569_b200.nsdgt import DGT_EILLEGAL_LENGTH, DGT_EINVAL, DgtError

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_remark_examples.txt")


def feasible(L, a, M, l1, l2):
    return L % a == 0 and L % M == 0 and (L // M) % l2 == 0 and (L // a) % l2 == 0


def lattice_set(gen, L):
    (a11, a12), (a21, a22) = gen
    pts = set()
    for i in range(L):
        for j in range(L):
            pts.add(((a11 * i + a12 * j) % L, (a21 * i + a22 * j) % L))
    return pts


def small_lattices(Lmax=72, l2max=4):
    for L in range(2, Lmax + 1):
        for a in range(1, L + 1):
            if L % a:
                continue
            for M in range(1, L + 1):
                if L % M:
                    continue
                for l2 in range(1, l2max + 1):
                    for l1 in range(0, l2):
                        if math.gcd(l1, l2) != 1 or not feasible(L, a, M, l1, l2):
                            continue
                        yield L, a, M, l1, l2


def test_golden_remark_examples():
    rows = [list(map(int, ln.split())) for ln in open(GOLDEN) if ln.strip() and not ln.startswith("#")]
    assert len(rows) == 2
    for a, M, l1, l2, c, Lmin, stride in rows:
        info = nsdgt.lattice_plan(Lmin, a, M, l1, l2)
        assert info["L_min"] == Lmin
        assert math.gcd(a, M) == c
        # the frequency shear can be avoided exactly at multiples of the printed stride
        for k in range(1, 3 * stride // Lmin + 1):
            L = k * Lmin
            branch = nsdgt.lattice_plan(L, a, M, l1, l2)["branch"]
            assert (branch == 1) == (L % stride == 0), (L, branch)


def test_minsig_bruteforce():
    """Prop. minsig: feasible lengths are exactly the multiples of lambda2 lcm(a,M)."""
    for a, M, l1, l2 in [(6, 6, 1, 2), (8, 12, 1, 2), (4, 6, 1, 3), (9, 12, 2, 3), (10, 4, 1, 4), (3, 5, 1, 2)]:
        Lmin = l2 * a * M // math.gcd(a, M)
        for L in range(1, 4 * Lmin + 1):
            ok = feasible(L, a, M, l1, l2)
            assert ok == (L % Lmin == 0)
            if ok:
                assert nsdgt.lattice_plan(L, a, M, l1, l2)["L_min"] == Lmin
            else:
                with pytest.raises(DgtError) as ei:
                    nsdgt.lattice_plan(L, a, M, l1, l2)
                assert ei.value.status == DGT_EILLEGAL_LENGTH
                assert ei.value.L_min == Lmin


def test_time_shear_existence_bruteforce():
    """A time-only shear is chosen iff some (0, s1) in Z_L^2 separates the lattice (brute force)."""
    for L, a, M, l1, l2 in small_lattices(Lmax=48, l2max=4):
        if l1 == 0:
            continue
        b = L // M
        s = b * l1 // l2
        exists = any(((s1 * a + s) % b) == 0 for s1 in range(L))
        info = nsdgt.lattice_plan(L, a, M, l1, l2)
        assert (info["branch"] == 1) == exists


def _check_identity(info):
    L, a, b, s = info["L"], info["a"], info["b"], info["s"]
    s0, s1 = info["s0"], info["s1"]
    Uinv = ((s0 * s1 + 1, s0), (s1, 1))
    A = ((a, 0), (s, b))
    prod = tuple(tuple(sum(Uinv[i][k] * A[k][j] for k in range(2)) % L for j in range(2)) for i in range(2))
    X = info["b_r"]
    D = ((a * b // X, 0), (0, X))
    assert lattice_set(prod, L) == lattice_set(D, L)
    # inner separable lattice of Algorithm 1 (time step, channels)
    if info["branch"] == 2:
        assert info["ia"] == X and info["iM"] == L // (a * b // X)
    else:
        assert info["ia"] == a and info["iM"] == info["M"]
    c, d, p, q = info["c"], info["d"], info["p"], info["q"]
    assert c * d * p * q == L and c == math.gcd(info["ia"], info["iM"])


@pytest.mark.parametrize("paper_shear", [False, True])
def test_shear_identity_all_small(paper_shear):
    """U^{-1} A Z_L^2 == D Z_L^2 (Eq. modcond satisfied) for every feasible lattice, L <= 48."""
    n = 0
    for L, a, M, l1, l2 in small_lattices(Lmax=48, l2max=4):
        info = nsdgt.lattice_plan(L, a, M, l1, l2, paper_shear=paper_shear)
        _check_identity(info)
        n += 1
    assert n > 500


def test_every_valid_s1_solves_modcond():
    """For each s1, the planner accepts the forced shear iff (modcond) is solvable; the
    accepted ones all satisfy the identity (sampled lattices up to L=96)."""
    for L, a, M, l1, l2 in [(36, 6, 6, 1, 3), (96, 8, 12, 1, 2), (72, 6, 8, 1, 3), (240, 8, 12, 1, 2)]:
        base = nsdgt.lattice_plan(L, a, M, l1, l2)
        b = base["b"]
        ok = 0
        for s1 in range(b):
            try:
                probe = nsdgt.lattice_plan(L, a, M, l1, l2, shear=(base["s0"], s1))
            except DgtError:
                probe = None
            if probe is not None:
                _check_identity(probe)
                ok += 1
        assert ok >= 1


def test_spec_examples():
    """Worked shear examples (derived by exhaustive search; SPEC.md:171-174 lists them)."""
    i = nsdgt.lattice_plan(16, 2, 4, 1, 2)
    assert (i["s0"], i["s1"], i["branch"]) == (0, 1, 1)
    i = nsdgt.lattice_plan(16, 4, 4, 1, 4)
    assert i["branch"] == 2 and i["s0"] != 0


def test_separable_and_errors():
    i = nsdgt.lattice_plan(36, 6, 6, 0, 1)
    assert i["branch"] == 0 and i["s0"] == 0 and i["s1"] == 0
    for bad in [(36, 6, 6, 1, 1), (36, 6, 6, 2, 4), (36, 0, 6, 0, 1), (36, 6, 6, -1, 2)]:
        with pytest.raises(DgtError) as ei:
            nsdgt.lattice_plan(*bad)
        assert ei.value.status == DGT_EINVAL
    with pytest.raises(DgtError):
        nsdgt.lattice_plan(36, 6, 6, 1, 3, shear=(1, 1))   # violates (modcond)


def test_baseline_configs_branches():
    """The policy picks the time shear where it exists and s1 = 0 for the frequency shear."""
    from synthetic import CONFIGS
    expect = {1: (2, 0), 2: (1, None), 3: (1, None), 4: (2, 0), 5: (1, None)}
    for wl in CONFIGS:
        info = nsdgt.lattice_plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2)
        br, s1 = expect[wl.k]
        assert info["branch"] == br
        if s1 is not None:
            assert info["s1"] == s1
        _check_identity(info) if wl.L <= 240 else None
        # inner shapes must be stageable on chip
        assert info["d"] <= 16384 and info["iM"] <= 16384
