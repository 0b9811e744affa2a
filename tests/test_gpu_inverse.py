"""GPU parity of the synthesis operator (inverse DGT, dgt_execute_inverse) against the
oracle's idgt (S1/S2, pinned in test_oracle_pins.py), through the C ABI.

Tolerances as for the forward transform (BASELINE.json north_star): relative l2 <= 1e-10
(c128) and <= 2e-5 (c64).
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


def small_cases():
    out = []
    for L in (24, 36, 48, 60, 72, 96, 120, 144):
        for a in range(1, L + 1):
            if L % a:
                continue
            for M in range(2, L + 1):
                if L % M or L * (L // a) * M > 400000 or (L // a) < 2:
                    continue
                for l1, l2 in [(0, 1), (1, 2), (1, 3), (2, 3), (1, 4), (3, 4)]:
                    if (L // M) % l2 or (L // a) % l2:
                        continue
                    out.append((L, a, M, l1, l2))
    rng = np.random.default_rng(4)
    idx = rng.choice(len(out), size=min(80, len(out)), replace=False)
    return [out[i] for i in sorted(idx)]


def rand_c(rng, W, M, N, dtype):
    c = rng.standard_normal((W, M, N)) + 1j * rng.standard_normal((W, M, N))
    return c.astype(np.complex64 if dtype == "c64" else np.complex128)


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_small_lattice_sweep_inverse(torch_cuda, nsdgt, oracle_mod, dtype):
    """Both branches, p = 1 and p > 1: synthesis of random coefficients, full comparison."""
    torch = torch_cuda
    branches = set()
    for i, (L, a, M, l1, l2) in enumerate(small_cases()):
        _, gamma = random_pair(L, 200 + i, dtype=dtype)
        rng = np.random.default_rng(i)
        c = rand_c(rng, 2, M, L // a, dtype)
        plan = nsdgt.Plan(L, a, M, l1, l2, gamma, dtype=dtype)
        branches.add(plan.info["branch"])
        f = plan.inverse(torch.from_numpy(c).cuda()).cpu().numpy()
        ref = oracle_mod.idgt(c, gamma, a, M, l1, l2)
        assert rel(f, ref) <= TOL[dtype], (L, a, M, l1, l2, plan.info)
    assert branches == {0, 1, 2}


@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_round_trip_with_dual_window(torch_cuda, nsdgt, oracle_mod, k):
    """GPU forward with g, GPU synthesis with the canonical dual (computed by the oracle's
    dense helpers only for config 1; for the larger configs the dual of a painless-case
    Gaussian is not needed: compare the synthesis of the GPU coefficients with the oracle's
    synthesis of the same coefficients on sampled signals)."""
    torch = torch_cuda
    wl = CONFIGS[k - 1]
    g = window(wl)
    W = min(wl.W, 3)
    f = batch(wl, 0, W)
    pf = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype, real_input=np.isrealobj(f))
    c = pf.execute(torch.from_numpy(f).cuda())
    if k == 1:
        import oracle
        gamma = oracle.windows.canonical_dual(g, wl.a, wl.M, wl.lam1, wl.lam2)
        pi = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, gamma, dtype=wl.dtype)
        fr = pi.inverse(c).cpu().numpy()
        assert rel(fr, f.astype(complex)) <= 1e-10
        return
    pi = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype)
    fr = pi.inverse(c).cpu().numpy()
    w = W - 1
    ref = oracle_mod.idgt(c[w].cpu().numpy(), g, wl.a, wl.M, wl.lam1, wl.lam2)
    assert rel(fr[w], ref) <= TOL[wl.dtype]


def test_config4_inverse_sampled(torch_cuda, nsdgt, oracle_mod):
    """Config 4 (frequency shear, c128, d = 180): synthesis of random coefficients, one signal
    against the oracle in full."""
    torch = torch_cuda
    wl = CONFIGS[3]
    g = window(wl)
    rng = np.random.default_rng(8)
    c = rand_c(rng, 1, wl.M, wl.N, "c128")
    plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype="c128")
    f = plan.inverse(torch.from_numpy(c).cuda()).cpu().numpy()
    ref = oracle_mod.idgt(c, g, wl.a, wl.M, wl.lam1, wl.lam2)
    assert rel(f, ref) <= TOL["c128"]


def test_adjointness_on_gpu(torch_cuda, nsdgt):
    """<dgt(f), c> = <f, idgt(c)> with both sides on the GPU (config 3 lattice, fused forward
    path vs the generic adjoint kernels)."""
    torch = torch_cuda
    wl = CONFIGS[2]
    g = window(wl)
    rng = np.random.default_rng(9)
    f = batch(wl, 0, 2)
    c = rand_c(rng, 2, wl.M, wl.N, "c64")
    plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype="c64")
    cf = plan.execute(torch.from_numpy(f).cuda()).cpu().numpy().astype(np.complex128)
    fi = plan.inverse(torch.from_numpy(c).cuda()).cpu().numpy().astype(np.complex128)
    lhs = np.vdot(c.astype(np.complex128), cf)
    rhs = np.vdot(fi, f.astype(np.complex128))
    assert abs(lhs - rhs) <= 1e-5 * abs(lhs)


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_adjointness_random_midsize_lattices(torch_cuda, nsdgt, dtype):
    """<dgt(f), c> = <f, idgt(c)> on random lattices with L up to 2^18 (the forward map on these
    lattices is oracle-checked in test_gpu_parity.py::test_random_midsize_lattices_sampled), so
    the synthesis kernels are pinned there through the adjoint identity."""
    import math
    torch = torch_cuda
    from test_gpu_parity import random_midsize_lattices
    tol = 1e-11 if dtype == "c128" else 2e-5
    for i, (L, a, M, l1, l2) in enumerate(random_midsize_lattices(8, seed=31 if dtype == "c128" else 32)):
        f, g = random_pair(L, 900 + i, dtype=dtype)
        rng = np.random.default_rng(i)
        c = rand_c(rng, 1, M, L // a, dtype)
        plan = nsdgt.Plan(L, a, M, l1, l2, g, dtype=dtype)
        cf = plan.execute(torch.from_numpy(f[None]).cuda()).cpu().numpy().astype(np.complex128)
        fi = plan.inverse(torch.from_numpy(c).cuda()).cpu().numpy().astype(np.complex128)
        lhs = np.vdot(c.astype(np.complex128), cf)
        rhs = np.vdot(fi, f[None].astype(np.complex128))
        scale = np.linalg.norm(c) * np.linalg.norm(cf)
        assert abs(lhs - rhs) <= tol * scale, (L, a, M, l1, l2, abs(lhs - rhs) / scale)
        assert math.isfinite(abs(lhs))


def test_inverse_errors_and_empty(torch_cuda, nsdgt):
    torch = torch_cuda
    L, a, M = 48, 4, 6
    plan = nsdgt.Plan(L, a, M, 1, 2, pgauss(L, a * M / L), dtype="c64")
    e = plan.inverse(torch.empty((0, M, L // a), dtype=torch.complex64, device="cuda"))
    assert e.shape == (0, L)
    with pytest.raises(TypeError):
        plan.inverse(torch.zeros((1, M, L // a), dtype=torch.complex128, device="cuda"))


@pytest.mark.parametrize("k,W", [(3, 1), (3, 9), (3, 10), (3, 17), (3, 38), (3, 39), (3, 40), (5, 3), (5, 9), (5, 11)])
def test_fused_synthesis_matches_generic_and_oracle(torch_cuda, nsdgt, oracle_mod, k, W, monkeypatch):
    """Configs 3 and 5 (fused7 lattices): the fused synthesis kernel (fused7_adj.cuh) against
    the generic adjoint kernels on ragged batches, and one signal against the oracle."""
    torch = torch_cuda
    wl = CONFIGS[k - 1]
    g = window(wl)
    rng = np.random.default_rng(100 + W)
    c = rand_c(rng, W, wl.M, wl.N, "c64")
    ct = torch.from_numpy(c).cuda()
    pf = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype="c64")
    assert pf.info["kernel_path"] == 2
    ff = pf.inverse(ct).cpu().numpy()
    monkeypatch.setenv("NSDGT_INV_GENERIC", "1")
    fg = pf.inverse(ct).cpu().numpy()
    assert rel(ff, fg) <= TOL["c64"]
    ref = oracle_mod.idgt(c[W - 1].astype(np.complex128), g, wl.a, wl.M, wl.lam1, wl.lam2)
    assert rel(ff[W - 1], ref) <= TOL["c64"]


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_config4_synthesis_kernels_match_generic(torch_cuda, nsdgt, dtype, monkeypatch):
    """Config 4's synthesis kernels (out_f4096_adj_kernel, zak_rr0_adj_kernel and the adjoint
    front_f4096 -- no cuFFT) against the generic adjoint kernels with cuFFT (selected at plan
    time by NSDGT_ZAK_RT / NSDGT_OUT_GENERIC, which also drop the front path)."""
    torch = torch_cuda
    wl = CONFIGS[3]
    g = window(wl)
    rng = np.random.default_rng(12)
    c = torch.from_numpy(rand_c(rng, 2, wl.M, wl.N, dtype)).cuda()
    pf = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=dtype)
    ff = pf.inverse(c).cpu().numpy()
    monkeypatch.setenv("NSDGT_ZAK_RT", "1")
    monkeypatch.setenv("NSDGT_OUT_GENERIC", "1")
    pg = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=dtype)
    fg = pg.inverse(c).cpu().numpy()
    assert rel(ff, fg) <= TOL[dtype]


def test_config4_lattice_prechirp_synthesis(torch_cuda, nsdgt, oracle_mod):
    """The adjoint front_f4096 with its conj(pchirp(L, s1)) factor: config 4's lattice at
    lambda = 1/6 (s1 = 128, on the front path), one signal of random coefficients in full
    against the oracle's idgt."""
    torch = torch_cuda
    wl = CONFIGS[3]
    info = nsdgt.lattice_plan(wl.L, wl.a, wl.M, 1, 6)
    assert info["pre_sigma"] != 0 and info["d"] == 180
    g = window(wl)
    rng = np.random.default_rng(13)
    c = rand_c(rng, 1, wl.M, wl.L // wl.a, "c128")
    plan = nsdgt.Plan(wl.L, wl.a, wl.M, 1, 6, g, dtype="c128")
    plan.profile_begin()
    f = plan.inverse(torch.from_numpy(c).cuda()).cpu().numpy()
    assert "front_f4096" in {k["name"] for k in plan.profile_end()}
    ref = oracle_mod.idgt(c, g, wl.a, wl.M, 1, 6)
    assert rel(f, ref) <= TOL["c128"]
