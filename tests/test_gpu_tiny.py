"""GPU parity of the one-CTA path (tiny.cuh: the whole shear algorithm of a short signal in one
CTA; Alg. 1, and its adjoint for the synthesis): every small lattice below is compared
in full with the oracle's dgt / idgt (both branches, p > q and p < q, separable lambda, real
input, both dtypes) and with the chunked kernels (NSDGT_TINY_OFF) of the same plan parameters."""
import numpy as np
import pytest

from synthetic import CONFIGS, batch, random_pair, window

pytestmark = pytest.mark.gpu
TOL = {"c64": 2e-5, "c128": 1e-10}

LATTICES = [  # (L, a, M, lambda1, lambda2)
    (48, 4, 6, 0, 1), (96, 8, 6, 0, 1), (96, 4, 6, 1, 2), (144, 6, 8, 1, 3), (240, 8, 12, 1, 2),
    (240, 8, 12, 1, 5), (360, 6, 12, 2, 3), (576, 8, 16, 1, 4), (720, 10, 12, 1, 6), (120, 12, 10, 1, 2),
    (240, 6, 20, 1, 4), (480, 24, 20, 1, 2),
]


def rel(x, y):
    return float(np.linalg.norm(x - y) / np.linalg.norm(y))


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import oracle
    import paper_1307_4569_b200 as nsdgt
    return torch, nsdgt, oracle


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("L,a,M,l1,l2", LATTICES)
def test_tiny_vs_oracle_and_chunked(env, dtype, L, a, M, l1, l2, monkeypatch):
    torch, nsdgt, oracle = env
    f, g = random_pair(L, 11 * L + l2, dtype=dtype)
    f2, _ = random_pair(L, 11 * L + l2 + 1, dtype=dtype)
    fb = torch.from_numpy(np.stack([f, f2])).cuda()
    plan = nsdgt.Plan(L, a, M, l1, l2, g, dtype=dtype)
    plan.profile_begin()
    c = plan.execute(fb)
    assert [k["name"] for k in plan.profile_end()] == ["tiny"]
    assert plan.launches(2) == 1
    assert rel(c.cpu().numpy(), oracle.dgt(np.stack([f, f2]), g, a, M, l1, l2)) <= TOL[dtype]
    # synthesis on the one-CTA path (tiny_adj_kernel) against the oracle's idgt
    plan.profile_begin()
    r = plan.inverse(c)
    assert [k["name"] for k in plan.profile_end()] == ["tiny_adjoint"]
    cn = c.cpu().numpy()
    assert rel(r.cpu().numpy(), oracle.idgt(cn, g, a, M, l1, l2)) <= TOL[dtype]
    monkeypatch.setenv("NSDGT_TINY_OFF", "1")
    p0 = nsdgt.Plan(L, a, M, l1, l2, g, dtype=dtype)
    c0 = p0.execute(fb)
    assert rel(c.cpu().numpy(), c0.cpu().numpy()) <= TOL[dtype]
    assert rel(r.cpu().numpy(), p0.inverse(c).cpu().numpy()) <= TOL[dtype]


def test_tiny_real_input_config1(env):
    """BASELINE config 1 (real fp64 f, frequency shear, p = 2) on the one-CTA path, W = 5."""
    torch, nsdgt, oracle = env
    wl = CONFIGS[0]
    g = window(wl)
    f = batch(wl, 0, 5)
    assert np.isrealobj(f)
    plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype="c128", real_input=True)
    c = plan.execute(torch.from_numpy(f).cuda()).cpu().numpy()
    assert rel(c, oracle.dgt(f, g, wl.a, wl.M, wl.lam1, wl.lam2)) <= 1e-10
    ch = plan.execute_host(f)
    assert np.array_equal(ch, c)


def test_tiny_many_signals_and_empty(env):
    """W = 0 launches nothing; W = 3000 short signals in one launch equal one-at-a-time runs."""
    torch, nsdgt, oracle = env
    L, a, M, l1, l2 = 144, 6, 8, 1, 3
    rng = np.random.default_rng(8)
    f = rng.standard_normal((3000, L)) + 1j * rng.standard_normal((3000, L))
    g = rng.standard_normal(L) + 1j * rng.standard_normal(L)
    plan = nsdgt.Plan(L, a, M, l1, l2, g, dtype="c128")
    assert plan.launches(0) == 0
    ft = torch.from_numpy(f).cuda()
    c = plan.execute(ft)
    for w in (0, 1777, 2999):
        assert torch.equal(c[w], plan.execute(ft[w:w + 1])[0])
    assert rel(c[1777].cpu().numpy(), oracle.dgt(f[1777], g, a, M, l1, l2)) <= 1e-10


@pytest.mark.parametrize("cfg", [0, 1, 3])
def test_input_produced_by_preceding_kernel(env, cfg):
    """The chunk kernels, front_f4096 and the one-CTA kernel are launched with programmatic
    dependent launch; each must wait for the preceding grid before reading the caller's input
    or writing anything.  Here a torch kernel writes f on the same stream right before every
    execute (and another reads the output right after): the results equal a fully
    synchronised run, repeated so that a missing wait would show."""
    torch, nsdgt, oracle = env
    wl = CONFIGS[cfg]
    g = window(wl)
    f0 = torch.from_numpy(batch(wl, 0, min(wl.W, 4))).cuda()
    plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype, real_input=wl.real_input)
    ref = []
    for k in range(3):
        fk = f0 * (k + 1) - 0.5 * k
        torch.cuda.synchronize()
        ref.append(plan.execute(fk).clone())
        torch.cuda.synchronize()
    fbuf = torch.empty_like(f0)
    out = torch.empty_like(ref[0])
    for rep in range(4):
        for k in range(3):
            torch.mul(f0, k + 1, out=fbuf)
            fbuf.sub_(0.5 * k)                   # f written by kernels right before the execute
            plan.execute(fbuf, out=out)
            got = out.clone()                    # read right after, same stream
            assert torch.equal(got, ref[k]), (rep, k)


def test_new_paths_bitwise_deterministic(env):
    """Shared-memory races in the round-2 kernels (one-CTA path, front_f4096, zak_rr0 and their
    adjoints, the config-2 output loads) would show as run-to-run differences: five runs of each
    are bit-for-bit equal (the library has no atomics and a fixed reduction order)."""
    torch, nsdgt, oracle = env
    for k in (0, 1, 3):
        wl = CONFIGS[k]
        g = window(wl)
        f = torch.from_numpy(batch(wl, 0, min(wl.W, 3))).cuda()
        plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype, real_input=wl.real_input)
        c0 = plan.execute(f).clone()
        r0 = plan.inverse(c0).clone()
        for _ in range(4):
            assert torch.equal(plan.execute(f), c0), wl.name
            assert torch.equal(plan.inverse(c0), r0), wl.name


@pytest.mark.parametrize("cfg", [0, 3])
def test_empty_batches_on_new_paths(env, cfg):
    """W = 0 on the one-CTA path (config 1) and on config 4's front path: forward, synthesis
    and the host path launch nothing and return empty results; a ragged batch (W not a multiple
    of the front batch / chunk) still matches signal-by-signal runs."""
    torch, nsdgt, oracle = env
    wl = CONFIGS[cfg]
    plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, window(wl), dtype=wl.dtype, real_input=wl.real_input)
    fdt = torch.float64 if wl.real_input else (torch.complex64 if wl.dtype == "c64" else torch.complex128)
    cdt = torch.complex64 if wl.dtype == "c64" else torch.complex128
    assert plan.launches(0) == 0
    e = plan.execute(torch.empty((0, wl.L), dtype=fdt, device="cuda"))
    assert e.shape == (0, wl.M, wl.N)
    r = plan.inverse(torch.empty((0, wl.M, wl.N), dtype=cdt, device="cuda"))
    assert r.shape[0] == 0
    W = 3 if cfg == 0 else 2
    f = torch.from_numpy(batch(wl, 0, W)).cuda()
    c = plan.execute(f)
    for w in range(W):
        assert torch.equal(c[w], plan.execute(f[w:w + 1])[0])
