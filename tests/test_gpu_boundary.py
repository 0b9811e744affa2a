"""Boundary contract checks on the GPU (include/nsdgt.h): dtype aliases in the binding, no
device allocation reachable from the execute entry points, and batches beyond the 65,535
grid-y limit of the chunked generic kernels."""
import numpy as np
import pytest

from synthetic import CONFIGS, batch, window

pytestmark = pytest.mark.gpu


def rel(x, y):
    return float(np.linalg.norm(x - y) / np.linalg.norm(y))


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import oracle
    import paper_1307_4569_b200 as nsdgt
    return torch, nsdgt, oracle


@pytest.mark.parametrize("alias,np_dt", [("complex64", np.complex64), ("fp32", np.complex64),
                                         ("complex128", np.complex128), ("float64", np.complex128)])
def test_dtype_aliases(env, alias, np_dt):
    """A plan made with a dtype alias returns arrays of that precision from the host path and
    the dual-window call (they were sized from the alias string before)."""
    torch, nsdgt, oracle = env
    L, a, M, l1, l2 = 480, 8, 12, 1, 2
    rng = np.random.default_rng(3)
    g = (rng.standard_normal(L) + 1j * rng.standard_normal(L)).astype(np_dt)
    f = (rng.standard_normal((2, L)) + 1j * rng.standard_normal((2, L))).astype(np_dt)
    plan = nsdgt.Plan(L, a, M, l1, l2, g, dtype=alias)
    assert plan.dtype in ("c64", "c128")
    c = plan.execute_host(f)
    assert c.dtype == np_dt and c.shape == (2, M, L // a)
    tol = 2e-5 if np_dt == np.complex64 else 1e-10
    assert rel(c, oracle.dgt(f, g, a, M, l1, l2)) <= tol
    gd = plan.dual_window()
    assert gd.dtype == np_dt
    assert rel(gd, oracle.windows.canonical_dual(g, a, M, l1, l2)) <= (1e-4 if np_dt == np.complex64 else 1e-9)


@pytest.mark.parametrize("k", [1, 3])
def test_execute_entry_points_allocate_nothing(env, k):
    """dgt_execute, dgt_execute_host and dgt_execute_inverse make no device allocation: the
    device's free memory is unchanged across calls with preallocated outputs (the plan made
    the chunk workspace, synthesis workspace and host staging)."""
    torch, nsdgt, _ = env
    wl = CONFIGS[k - 1]
    W = 3
    f = batch(wl, 0, W)
    plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, window(wl), dtype=wl.dtype, real_input=wl.real_input)
    cdt = torch.complex64 if wl.dtype == "c64" else torch.complex128
    fd = torch.from_numpy(f).cuda()
    cd = torch.empty((W, wl.M, wl.N), dtype=cdt, device="cuda")
    fo = torch.empty((W, wl.L), dtype=cdt, device="cuda")
    fh = torch.from_numpy(f).pin_memory()
    ch = torch.empty((W, wl.M, wl.N), dtype=cdt).pin_memory()
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(2):
        plan.execute(fd, out=cd)
        plan.inverse(cd, out=fo)
        plan.execute_host(fh, out=ch)
    torch.cuda.synchronize()
    assert torch.cuda.mem_get_info()[0] == free0
    assert np.array_equal(ch.numpy(), cd.cpu().numpy())


def test_batch_beyond_grid_y_limit(env):
    """Config 1's lattice (generic kernels, chunked) with W = 70,000 > 65,535 signals: the
    chunk is bounded, every chunk runs, sampled signals match the oracle."""
    torch, nsdgt, oracle = env
    wl = CONFIGS[0]
    W = 70000
    g = window(wl)
    rng = np.random.default_rng(5)
    f = rng.standard_normal((W, wl.L))
    plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype="c128", real_input=True)
    assert plan.info["chunk"] <= 65535
    c = plan.execute(torch.from_numpy(f).cuda())
    ws = np.array([0, 8191, 8192, 65535, 65536, W - 1])
    got = c[torch.from_numpy(ws).cuda()].cpu().numpy()
    ref = oracle.dgt(f[ws], g, wl.a, wl.M, wl.lam1, wl.lam2, variant="literal")
    assert rel(got, ref) <= 1e-10
