"""GPU parity of the fused7 hot-path kernel (csrc/fused7.cuh).

fused7 serves time-shear / separable lattices with p = 1, q = 4, d = M in {256, 512}
(BASELINE configs 3 and 5).  Its job queue, ring of intermediate slots and look-ahead depend
on W, so these tests sweep small and ragged batch sizes (W below the look-ahead, W = 1),
other valid shears (sigma_j != 0: the shifted gather), the separable lattice, and compare
with the oracle on sampled columns and with the generic kernels (themselves oracle-checked)
on every coefficient.  Tolerance: north_star's 2e-5 relative l2 for complex64.
"""
import numpy as np
import pytest

from synthetic import CONFIGS, window

pytestmark = pytest.mark.gpu
TOL = 2e-5


def rel(x, y):
    return float(np.linalg.norm(x - y) / np.linalg.norm(y))


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import oracle
    import paper_1307_4569_b200 as nsdgt
    return torch, nsdgt, oracle


def signals(L, W, seed):
    rng = np.random.default_rng(seed)
    return ((rng.standard_normal((W, L)) + 1j * rng.standard_normal((W, L))) / np.sqrt(2)).astype(np.complex64)


def check(env, L, a, M, l1, l2, g, W, seed, shear=None, expect_fused=True, ncols=24):
    torch, nsdgt, oracle = env
    f = signals(L, W, seed)
    plan = nsdgt.Plan(L, a, M, l1, l2, g, dtype="c64", shear=shear)
    if expect_fused:
        assert plan.info["kernel_path"] == 2, plan.info
    ref_plan = nsdgt.Plan(L, a, M, l1, l2, g, dtype="c64", shear=shear, force_generic=True)
    assert ref_plan.info["kernel_path"] == 0
    ft = torch.from_numpy(f).cuda()
    c = plan.execute(ft).cpu().numpy()
    cg = ref_plan.execute(ft).cpu().numpy()
    assert c.shape == (W, M, L // a)
    assert rel(c, cg) <= TOL, ("vs generic", W)
    rng = np.random.default_rng(seed + 1)
    ws = sorted(set([0, W - 1] + list(rng.choice(W, min(W, 2), replace=False))))
    cols = np.sort(rng.choice(L // a, ncols, replace=False))
    ref = oracle.dgt(f[ws], g, a, M, l1, l2, cols=cols)
    assert rel(c[ws][:, :, cols], ref) <= TOL, ("vs oracle", W)
    return plan


@pytest.mark.parametrize("W", [1, 2, 3, 5, 17, 23, 24, 38, 39, 40, 77])
def test_config3_lattice_small_and_ragged_batches(env, W):
    """W below, at and above the look-ahead (23) and the ring size (38) of config 3's plan."""
    wl = CONFIGS[2]
    check(env, wl.L, wl.a, wl.M, wl.lam1, wl.lam2, window(wl), W, seed=100 + W)


@pytest.mark.parametrize("W", [1, 3, 9])
def test_config5_lattice_small_batches(env, W):
    wl = CONFIGS[4]
    check(env, wl.L, wl.a, wl.M, wl.lam1, wl.lam2, window(wl), W, seed=200 + W, ncols=12)


def test_separable_lattice(env):
    """lambda = 0: s1 = 0, no chirp, no rotation, E = 1."""
    wl = CONFIGS[2]
    plan = check(env, wl.L, wl.a, wl.M, 0, 1, window(wl), 6, seed=301)
    assert plan.info["s1"] == 0


def test_other_valid_time_shears(env):
    """Every valid time shear s1 of config 3's lattice gives the same c (reading Z9).  Other
    s1 change the chirp rate K and the rotation slope beta that fused7 folds into G' (in
    fused7's domain d = b = M, so sigma_j = (j beta - K j) mod D is always 0)."""
    torch, nsdgt, oracle = env
    wl = CONFIGS[2]
    g = window(wl)
    seen = 0
    for s1 in range(0, 2 * wl.M):
        try:
            info = nsdgt.lattice_plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, shear=(0, s1))
        except nsdgt.DgtError:
            continue
        if info["branch"] != 1 or info["p"] != 1 or info["d"] != wl.M:
            continue
        plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype="c64", shear=(0, s1))
        if plan.info["kernel_path"] != 2:
            continue
        check(env, wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, 3, seed=400 + s1, shear=(0, s1), ncols=8)
        seen += 1
        if seen >= 4:
            break
    assert seen >= 2, "expected several valid time shears served by fused7"


def test_delta_window_closed_form_fused7(env):
    """g = delta_0 => c(m, n) = f(a n) exp(-2 pi i (m + w(n)) a n / M) (pin P3), every coefficient."""
    torch, nsdgt, oracle = env
    wl = CONFIGS[2]
    g = np.zeros(wl.L, dtype=np.complex64)
    g[0] = 1
    W = 4
    f = signals(wl.L, W, 501)
    plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype="c64")
    assert plan.info["kernel_path"] == 2
    c = plan.execute(torch.from_numpy(f).cuda()).cpu().numpy()
    m = np.arange(wl.M)[:, None]
    n = np.arange(wl.N)[None, :]
    num = ((m * wl.lam2 + (n * wl.lam1) % wl.lam2) * wl.a * n) % (wl.lam2 * wl.M)
    ph = np.exp(-2j * np.pi * num / (wl.lam2 * wl.M))
    for w in range(W):
        assert rel(c[w], f[w][wl.a * n].astype(np.complex128) * ph) <= TOL


def test_repeat_execute_deterministic(env):
    """The dynamic job queue must not change results: two executes are bitwise equal."""
    torch, nsdgt, oracle = env
    wl = CONFIGS[2]
    f = torch.from_numpy(signals(wl.L, 33, 601)).cuda()
    plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, window(wl), dtype="c64")
    c1 = plan.execute(f)
    c2 = plan.execute(f)
    assert torch.equal(c1, c2)


def test_real_input_on_fused_lattice(env):
    """A real-input plan on config 3's lattice (fused7 promotes real samples on load) matches the
    oracle and the complex-input fused plan."""
    torch, nsdgt, oracle = env
    wl = CONFIGS[2]
    g = window(wl)
    f = np.random.default_rng(11).standard_normal((2, wl.L)).astype(np.float32)
    pr = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype="c64", real_input=True)
    assert pr.info["kernel_path"] == 2
    cr = pr.execute(torch.from_numpy(f).cuda()).cpu().numpy()
    pc = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype="c64")
    cc = pc.execute(torch.from_numpy(f.astype(np.complex64)).cuda()).cpu().numpy()
    assert rel(cr, cc) <= TOL
    cols = np.arange(0, wl.N, 97)
    assert rel(cr[:, :, cols], oracle.dgt(f, g, wl.a, wl.M, wl.lam1, wl.lam2, cols=cols)) <= TOL


def test_shard_results_bitwise_equal(env):
    """SURVEY §4 T6 on one GPU: a batch split into shards (what each rank of a multi-GPU run
    transforms) gives bit-for-bit the coefficients of the whole batch -- the per-signal
    arithmetic does not depend on W or on the ring slot."""
    torch, nsdgt, _ = env
    for k, W in ((5, 8), (3, 40)):
        wl = CONFIGS[k - 1]
        plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, window(wl), dtype="c64")
        ft = torch.from_numpy(signals(wl.L, W, 900 + k)).cuda()
        whole = plan.execute(ft)
        parts = [plan.execute(ft[i:i + W // 4].contiguous()) for i in range(0, W, W // 4)]
        assert torch.equal(whole, torch.cat(parts)), k
