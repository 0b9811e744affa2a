"""GPU canonical dual / tight windows (dgt_window_dual) against the oracle's
dense frame operator (oracle/windows.py, pinned in test_oracle_pins.py), and GPU perfect
reconstruction at the BASELINE configs' full sizes.

Tolerances: relative l2 <= 1e-10 (c128), <= 2e-5 (c64), as for the transform.
"""
import numpy as np
import pytest

from synthetic import CONFIGS, batch, pgauss, random_pair, window

pytestmark = pytest.mark.gpu

TOL = {"c64": 2e-5, "c128": 1e-10}


def rel(x, y):
    return float(np.linalg.norm(x - y) / np.linalg.norm(y))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


@pytest.fixture(scope="module")
def nsdgt():
    import paper_1307_4569_b200 as m
    return m


# both branches, p = 1 and p = 2 (config 1), separable, lambda2 up to 4; redundancy > 1
LATTICES = [(240, 8, 12, 1, 2), (72, 8, 12, 1, 3), (36, 6, 12, 1, 3), (96, 8, 12, 1, 4), (120, 10, 12, 0, 1),
            (144, 12, 18, 1, 2), (216, 12, 18, 1, 3), (480, 16, 24, 1, 2), (360, 20, 30, 2, 3), (288, 8, 16, 1, 3)]


@pytest.mark.parametrize("L,a,M,l1,l2", LATTICES)
@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_dual_and_tight_vs_dense(nsdgt, oracle_mod, L, a, M, l1, l2, dtype):
    g = pgauss(L, a * M / L)
    plan = nsdgt.Plan(L, a, M, l1, l2, g, dtype=dtype)
    gd = plan.dual_window()
    assert rel(gd, oracle_mod.windows.canonical_dual(g, a, M, l1, l2)) <= TOL[dtype], plan.info
    if plan.info["p"] <= 2:
        gt = plan.dual_window(tight=True)
        assert rel(gt, oracle_mod.windows.canonical_tight(g, a, M, l1, l2)) <= TOL[dtype], plan.info


def test_random_window_dual(nsdgt, oracle_mod):
    """A non-symmetric complex window (no Gaussian structure) on a frequency-shear lattice."""
    L, a, M, l1, l2 = 72, 8, 12, 1, 3
    _, g = random_pair(L, 51)
    plan = nsdgt.Plan(L, a, M, l1, l2, g, dtype="c128")
    assert rel(plan.dual_window(), oracle_mod.windows.canonical_dual(g, a, M, l1, l2)) <= 1e-10


@pytest.mark.parametrize("k", [2, 3, 4, 5])
def test_perfect_reconstruction_full_size(torch_cuda, nsdgt, k):
    """BASELINE configs at full size: gamma = GPU dual of g; GPU synthesis of the GPU analysis
    coefficients with gamma returns f (the inversion formula)."""
    torch = torch_cuda
    wl = CONFIGS[k - 1]
    g = window(wl)
    W = 2
    f = batch(wl, 0, W)
    pa = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype)
    gamma = pa.dual_window()
    ps = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, gamma, dtype=wl.dtype)
    fr = ps.inverse(pa.execute(torch.from_numpy(f).cuda())).cpu().numpy()
    assert rel(fr, f) <= (1e-9 if wl.dtype == "c128" else 5e-5)


def test_tight_window_parseval_full_size(torch_cuda, nsdgt):
    """Config 3: the GPU tight window gives a Parseval frame: ||c||^2 = ||f||^2 and synthesis with
    the same window reconstructs f."""
    torch = torch_cuda
    wl = CONFIGS[2]
    g = window(wl)
    pt = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype="c64")
    gt = pt.dual_window(tight=True)
    p2 = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, gt, dtype="c64")
    f = batch(wl, 0, 2)
    c = p2.execute(torch.from_numpy(f).cuda())
    ratio = float((c.abs() ** 2).sum().item() / np.sum(np.abs(f) ** 2))
    assert abs(ratio - 1.0) < 1e-4
    assert rel(p2.inverse(c).cpu().numpy(), f) <= 5e-5
