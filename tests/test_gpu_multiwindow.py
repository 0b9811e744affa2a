"""GPU parity of the multiwindow algorithm (dgt_plan_multiwindow, PAPER.md:344-420,
Prop. mwindec and Eq. mw_phases): the same transform Eq. (DGT) as the shear plans, computed as
lambda2 separable DGTs on (lambda2 a, b) with the windows g_m = M_{m s mod b} T_{m a} g joined by
phase factors.  Compared in full with the oracle on small lattices (both dtypes, real input,
lambda2 = 1 .. 6), with the shear plan on every coefficient of the Fig. 2 lattices, and on
sampled columns with the oracle there."""
import math

import numpy as np
import pytest

from synthetic import random_pair

pytestmark = pytest.mark.gpu
TOL = {"c64": 2e-5, "c128": 1e-10}


def rel(x, y):
    return float(np.linalg.norm(x - y) / np.linalg.norm(y))


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import oracle
    import paper_1307_4569_b200 as nsdgt
    return torch, nsdgt, oracle


SMALL = [  # (L, a, M, lambda1, lambda2)
    (48, 4, 6, 0, 1), (96, 4, 6, 1, 2), (144, 6, 8, 1, 3), (240, 8, 12, 1, 2), (240, 8, 12, 1, 5),
    (360, 6, 12, 2, 3), (576, 8, 16, 1, 4), (720, 10, 12, 1, 6), (4096, 64, 256, 1, 2),
]


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("L,a,M,l1,l2", SMALL)
def test_small_lattices_vs_oracle(env, dtype, L, a, M, l1, l2):
    torch, nsdgt, oracle = env
    f, g = random_pair(L, 7 * L + l2, dtype=dtype)
    f2, _ = random_pair(L, 7 * L + l2 + 1, dtype=dtype)
    fb = np.stack([f, f2])
    plan = nsdgt.Plan(L, a, M, l1, l2, g, dtype=dtype, algorithm="multiwindow")
    assert plan.info["kernel_path"] >= 32
    c = plan.execute(torch.from_numpy(fb).cuda()).cpu().numpy()
    assert rel(c, oracle.dgt(fb, g, a, M, l1, l2)) <= TOL[dtype]


def test_real_input(env):
    torch, nsdgt, oracle = env
    L, a, M, l1, l2 = 240, 8, 12, 1, 2
    rng = np.random.default_rng(4)
    f = rng.standard_normal((3, L))
    g = rng.standard_normal(L) + 1j * rng.standard_normal(L)
    plan = nsdgt.Plan(L, a, M, l1, l2, g, dtype="c128", real_input=True, algorithm="multiwindow")
    c = plan.execute(torch.from_numpy(f).cuda()).cpu().numpy()
    assert rel(c, oracle.dgt(f, g, a, M, l1, l2)) <= 1e-10
    # host path and chunking: execute_host equals execute bit for bit
    ch = plan.execute_host(f)
    assert np.array_equal(ch, c)


@pytest.mark.parametrize("a,M", [(32, 64), (40, 60), (60, 80)])
@pytest.mark.parametrize("lam2", [2, 3, 5])
def test_fig2_lattices_equal_shear(env, a, M, lam2):
    """The Fig. 2 lattices (L = lcm(a, M) 2520, lambda = 1/lambda2): multiwindow and shear plans
    agree on every coefficient of two signals; sampled columns against the oracle."""
    torch, nsdgt, oracle = env
    from synthetic import pgauss
    L = a * M // math.gcd(a, M) * 2520
    g = pgauss(L, a * M / L).astype(np.complex64)
    f = np.stack([random_pair(L, 90 + lam2, dtype="c64")[0], random_pair(L, 91 + lam2, dtype="c64")[0]])
    ft = torch.from_numpy(f).cuda()
    cm = nsdgt.Plan(L, a, M, 1, lam2, g, dtype="c64", algorithm="multiwindow").execute(ft).cpu().numpy()
    cs = nsdgt.Plan(L, a, M, 1, lam2, g, dtype="c64").execute(ft).cpu().numpy()
    assert rel(cm, cs) <= 2 * TOL["c64"]
    cols = np.sort(np.random.default_rng(lam2).choice(L // a, 8, replace=False))
    ref = oracle.dgt(f[:1], g, a, M, 1, lam2, cols=cols)
    assert rel(cm[:1][:, :, cols], ref) <= TOL["c64"]


def test_unsupported_entry_points(env):
    torch, nsdgt, _ = env
    L, a, M, l1, l2 = 96, 4, 6, 1, 2
    _, g = random_pair(L, 3, dtype="c64")
    plan = nsdgt.Plan(L, a, M, l1, l2, g, dtype="c64", algorithm="multiwindow")
    c = torch.zeros((1, M, L // a), dtype=torch.complex64, device="cuda")
    with pytest.raises(nsdgt.DgtError) as e:
        plan.inverse(c)
    assert e.value.status == nsdgt.DGT_EUNSUPPORTED
    with pytest.raises(nsdgt.DgtError) as e:
        plan.dual_window()
    assert e.value.status == nsdgt.DGT_EUNSUPPORTED
