"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerances (BASELINE.json north_star): relative l2 error <= 1e-10 for fp64 (c128) and
<= 2e-5 for fp32 (c64), over the compared coefficients.  Small lattices are compared
element by element in full; BASELINE.json's configs run at full size in bench.py's
launch configuration (full W, default chunking) and are compared on sampled signals /
columns the oracle computes one by one.
"""
import math

import numpy as np
import pytest

from synthetic import CONFIGS, batch, random_pair, window

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


def run_gpu(nsdgt, torch, f, g, L, a, M, l1, l2, dtype, **kw):
    plan = nsdgt.Plan(L, a, M, l1, l2, g, dtype=dtype, real_input=np.isrealobj(f), **kw)
    ft = torch.from_numpy(np.ascontiguousarray(f)).cuda()
    c = plan.execute(ft)
    torch.cuda.synchronize()
    return c.cpu().numpy(), plan


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
    rng = np.random.default_rng(3)
    idx = rng.choice(len(out), size=min(120, len(out)), replace=False)
    return [out[i] for i in sorted(idx)]


SMALL = small_cases()


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_small_lattice_sweep(torch_cuda, nsdgt, oracle_mod, dtype):
    """Feasible lattices L <= 144 (both branches, p = 1 and p > 1), full comparison."""
    worst = 0.0
    branches = set()
    for i, (L, a, M, l1, l2) in enumerate(SMALL):
        f, g = random_pair(L, 100 + i, dtype=dtype)
        c, plan = run_gpu(nsdgt, torch_cuda, f, g, L, a, M, l1, l2, dtype)
        branches.add(plan.info["branch"])
        ref = oracle_mod.dgt(f, g, a, M, l1, l2, variant="literal")
        e = rel(c, ref)
        worst = max(worst, e)
        assert e <= TOL[dtype], (L, a, M, l1, l2, plan.info, e)
    assert branches == {0, 1, 2}


@pytest.mark.parametrize("L,a,M,l1,l2", [(36, 6, 6, 1, 3), (96, 8, 12, 1, 2), (72, 6, 8, 1, 3), (240, 8, 12, 1, 2),
                                         (160, 10, 8, 1, 4)])
def test_every_valid_shear_same_c(torch_cuda, nsdgt, oracle_mod, L, a, M, l1, l2):
    """Every (s0, s1) satisfying Eq. (modcond) gives the same c (reading Z9), incl. the
    paper's own s1 choice (Eq. s1choice)."""
    f, g = random_pair(L, 7, dtype="c128")
    ref = oracle_mod.dgt(f, g, a, M, l1, l2, variant="literal")
    base = nsdgt.lattice_plan(L, a, M, l1, l2)
    tried = 0
    for s1 in range(base["b"]):
        shear = None
        for s0 in range(L):
            try:
                nsdgt.lattice_plan(L, a, M, l1, l2, shear=(s0, s1))
                shear = (s0, s1)
                break
            except nsdgt.DgtError:
                continue
        if shear is None:
            continue
        c, plan = run_gpu(nsdgt, torch_cuda, f, g, L, a, M, l1, l2, "c128", shear=shear)
        assert rel(c, ref) <= 1e-10, (shear, plan.info)
        tried += 1
    c, _ = run_gpu(nsdgt, torch_cuda, f, g, L, a, M, l1, l2, "c128", paper_shear=True)
    assert rel(c, ref) <= 1e-10
    assert tried >= 1


def test_real_input_config1(torch_cuda, nsdgt, oracle_mod):
    """Config 1 exactly as in BASELINE.json: real fp64 f, pgauss window, frequency shear."""
    wl = CONFIGS[0]
    f = batch(wl, 0, wl.W)
    g = window(wl)
    c, plan = run_gpu(nsdgt, torch_cuda, f, g, wl.L, wl.a, wl.M, wl.lam1, wl.lam2, wl.dtype)
    assert plan.info["branch"] == 2 and plan.info["p"] == 2
    ref = oracle_mod.dgt(f, g, wl.a, wl.M, wl.lam1, wl.lam2, variant="literal")
    assert rel(c, ref) <= 1e-10


@pytest.mark.parametrize("k", [2, 3, 4, 5])
def test_baseline_config_full_size(torch_cuda, nsdgt, oracle_mod, k):
    """BASELINE configs at full size and full W (bench.py's launch configuration).
    Whole signals are compared for a few w (config 4: signal 0 in full, all 12,288 columns x
    240 channels against the regrouped oracle, plus sampled columns of the last signal);
    every other w is compared on sampled columns."""
    wl = CONFIGS[k - 1]
    torch = torch_cuda
    g = window(wl)
    f = batch(wl, 0, wl.W)
    plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype)
    c = plan.execute(torch.from_numpy(f).cuda())
    torch.cuda.synchronize()
    rng = np.random.default_rng(k)
    full_ws = [0, wl.W - 1]
    for w in sorted(set(full_ws)):
        if k == 4 and w > 0:
            cols = np.sort(rng.choice(wl.N, 96, replace=False))
            ref = oracle_mod.dgt(f[w], g, wl.a, wl.M, wl.lam1, wl.lam2, cols=cols)
            got = c[w][:, torch.from_numpy(cols).cuda()].cpu().numpy()
        else:
            ref = oracle_mod.dgt(f[w], g, wl.a, wl.M, wl.lam1, wl.lam2)
            got = c[w].cpu().numpy()
        assert rel(got, ref) <= TOL[wl.dtype], (k, w)
    # sampled signals x sampled columns
    ws = np.sort(rng.choice(wl.W, min(wl.W, 6), replace=False))
    cols = np.sort(rng.choice(wl.N, 8, replace=False))
    ref = oracle_mod.dgt(f[ws], g, wl.a, wl.M, wl.lam1, wl.lam2, cols=cols)
    got = c[torch.from_numpy(ws).cuda()][:, :, torch.from_numpy(cols).cuda()].cpu().numpy()
    assert rel(got, ref) <= TOL[wl.dtype]


@pytest.mark.parametrize("k", [3, 5])
def test_delta_window_full_size(torch_cuda, nsdgt, k):
    """Full-size invariant (no oracle): g = delta_0 => c(m,n) = f(an) e^{-2 pi i (m+w(n)) a n / M}."""
    wl = CONFIGS[k - 1]
    torch = torch_cuda
    g = np.zeros(wl.L, dtype=np.complex64 if wl.dtype == "c64" else np.complex128)
    g[0] = 1
    W = 8
    f = batch(wl, 0, W)
    plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype)
    c = plan.execute(torch.from_numpy(f).cuda()).cpu().numpy()
    m = np.arange(wl.M)[:, None]
    n = np.arange(wl.N)[None, :]
    num = ((m * wl.lam2 + (n * wl.lam1) % wl.lam2) * wl.a * n) % (wl.lam2 * wl.M)
    ph = np.exp(-2j * np.pi * num / (wl.lam2 * wl.M))
    for w in range(W):
        ref = f[w][wl.a * n].astype(np.complex128) * ph
        assert rel(c[w], ref) <= TOL[wl.dtype]


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_fbranch_out4096_kernel(torch_cuda, nsdgt, oracle_mod, dtype, monkeypatch):
    """Frequency shear with N_r = 4096 inner channels takes the out_f4096 kernel (config 4's
    output kernel): full comparison on a lattice the oracle finishes in seconds, and
    agreement with the generic Stockham output kernel."""
    torch = torch_cuda
    L, a, M, l1, l2 = 36864, 3, 12, 1, 3
    info = nsdgt.lattice_plan(L, a, M, l1, l2)
    assert info["branch"] == 2 and info["iM"] == 4096
    f, g = random_pair(L, 41, dtype=dtype)
    f2, _ = random_pair(L, 42, dtype=dtype)
    fb = np.stack([f, f2])
    c, _ = run_gpu(nsdgt, torch, fb, g, L, a, M, l1, l2, dtype)
    ref = oracle_mod.dgt(fb, g, a, M, l1, l2)
    assert rel(c, ref) <= TOL[dtype]
    monkeypatch.setenv("NSDGT_OUT_GENERIC", "1")
    cg, _ = run_gpu(nsdgt, torch, fb, g, L, a, M, l1, l2, dtype)
    assert rel(c, cg) <= TOL[dtype]


def test_config4_lattice_c64_sampled(torch_cuda, nsdgt, oracle_mod):
    """Config 4's lattice in complex64 (the d = 180 Zak kernel's 8-column variant and
    out_f4096 in fp32): sampled columns of two signals against the oracle."""
    torch = torch_cuda
    wl = CONFIGS[3]
    g = window(wl).astype(np.complex64)
    f = batch(wl, 0, 2).astype(np.complex64)
    plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype="c64")
    c = plan.execute(torch.from_numpy(f).cuda())
    cols = np.sort(np.random.default_rng(44).choice(wl.N, 24, replace=False))
    ref = oracle_mod.dgt(f, g, wl.a, wl.M, wl.lam1, wl.lam2, cols=cols)
    got = c[:, :, torch.from_numpy(cols).cuda()].cpu().numpy()
    assert rel(got, ref) <= TOL["c64"]


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_config4_front_and_zak_variants_agree(torch_cuda, nsdgt, oracle_mod, dtype, monkeypatch):
    """Config 4 runs front_f4096 + zak_rr0 (the length-L FFT split as 4096-point DFTs of the
    180 residues and a DFT_180 inside the Zak kernel; no cuFFT).  The same plan with cuFFT's
    front end + zak_rr (NSDGT_FRONT_CUFFT) and with cuFFT + the Stockham zak_ct (also
    NSDGT_ZAK_CT) agree with it and with the oracle on sampled columns; the synthesis
    (zak_rr0_adj + the adjoint front) agrees with cuFFT + zak_ct_adj."""
    torch = torch_cuda
    wl = CONFIGS[3]
    g = window(wl)
    fnp = batch(wl, 0, 2).astype(np.complex64 if dtype == "c64" else np.complex128)
    f = torch.from_numpy(fnp).cuda()
    p = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=dtype)
    p.profile_begin()
    c = p.execute(f)
    names = {k["name"] for k in p.profile_end()}
    assert "front_f4096" in names and "front_fft_cufft" not in names, names
    # synthesis: zak_rr0_adj + the adjoint front_f4096 (no cuFFT) against cuFFT + zak_ct_adj
    rsyn = p.inverse(c)
    monkeypatch.setenv("NSDGT_FRONT_CUFFT", "1")
    p1 = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=dtype)
    c1 = p1.execute(f)
    rsyn1 = p1.inverse(c)
    monkeypatch.setenv("NSDGT_ZAK_CT", "1")
    c2 = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=dtype).execute(f)
    tol = TOL[dtype]
    assert rel(c.cpu().numpy(), c1.cpu().numpy()) <= tol
    assert rel(c.cpu().numpy(), c2.cpu().numpy()) <= tol
    assert rel(rsyn.cpu().numpy(), rsyn1.cpu().numpy()) <= tol
    cols = np.sort(np.random.default_rng(45).choice(wl.N, 16, replace=False))
    ref = oracle_mod.dgt(fnp, g, wl.a, wl.M, wl.lam1, wl.lam2, cols=cols)
    assert rel(c[:, :, torch.from_numpy(cols).cuda()].cpu().numpy(), ref) <= tol


@pytest.mark.parametrize("lam", [(1, 3), (1, 6)])
def test_front_f4096_real_input_and_prechirp(torch_cuda, nsdgt, oracle_mod, lam):
    """front_f4096's real-input load and its pchirp(L, s1) multiplier: config 4's lattice with
    real f (lambda = 1/3, s1 = 0) and lambda = 1/6 (s1 = 128, the pre-chirp), both on the
    front_f4096 path, sampled columns against the oracle."""
    torch = torch_cuda
    wl = CONFIGS[3]
    l1, l2 = lam
    info = nsdgt.lattice_plan(wl.L, wl.a, wl.M, l1, l2)
    assert info["d"] == 180 and info["c"] * info["q"] == 4096
    g = window(wl)
    fc = batch(wl, 0, 1)
    f = np.ascontiguousarray(fc.real) if lam == (1, 3) else fc
    if lam == (1, 6):
        assert info["pre_sigma"] != 0
    p = nsdgt.Plan(wl.L, wl.a, wl.M, l1, l2, g, dtype="c128", real_input=np.isrealobj(f))
    p.profile_begin()
    c = p.execute(torch.from_numpy(f).cuda())
    assert "front_f4096" in {k["name"] for k in p.profile_end()}
    N = wl.L // wl.a
    cols = np.sort(np.random.default_rng(46).choice(N, 12, replace=False))
    ref = oracle_mod.dgt(f, g, wl.a, wl.M, l1, l2, cols=cols)
    assert rel(c[:, :, torch.from_numpy(cols).cuda()].cpu().numpy(), ref) <= TOL["c128"]


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_config4_intermediate_layouts_bitwise_equal(torch_cuda, nsdgt, dtype, monkeypatch):
    """zak_ct -> out_f4096 on config 4 store the intermediate [n][j] (contiguous output-kernel
    loads); the generic [j][kappa][n'] layout (NSDGT_CNJ_OFF) runs the same arithmetic, so
    analysis and synthesis are bit-for-bit equal between the two layouts."""
    torch = torch_cuda
    wl = CONFIGS[3]
    g = window(wl)
    f = torch.from_numpy(batch(wl, 0, 3).astype(np.complex64 if dtype == "c64" else np.complex128)).cuda()
    p1 = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=dtype)
    c1 = p1.execute(f)
    r1 = p1.inverse(c1)
    monkeypatch.setenv("NSDGT_CNJ_OFF", "1")
    p0 = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=dtype)
    c0 = p0.execute(f)
    r0 = p0.inverse(c0)
    assert torch.equal(c1, c0)
    assert torch.equal(r1, r0)


def test_chunking_ragged_and_host_path(torch_cuda, nsdgt):
    """Ragged chunks (W not a multiple of the chunk), W = 0, and the host end-to-end path
    give bitwise the same result as one device execute."""
    torch = torch_cuda
    L, a, M, l1, l2 = 4096, 32, 64, 1, 2
    rng = np.random.default_rng(9)
    W = 7
    f = (rng.standard_normal((W, L)) + 1j * rng.standard_normal((W, L))).astype(np.complex64)
    _, g = random_pair(L, 3, dtype="c64")
    p1 = nsdgt.Plan(L, a, M, l1, l2, g, dtype="c64")
    p3 = nsdgt.Plan(L, a, M, l1, l2, g, dtype="c64", max_chunk=3)
    ft = torch.from_numpy(f).cuda()
    c1 = p1.execute(ft).cpu().numpy()
    c3 = p3.execute(ft).cpu().numpy()
    assert np.array_equal(c1, c3)
    ch = p3.execute_host(f)
    assert np.array_equal(ch, c1)
    pinned = torch.from_numpy(f).pin_memory()
    ch2 = p3.execute_host(pinned)
    assert np.array_equal(ch2.numpy(), c1)
    empty = p1.execute(torch.empty((0, L), dtype=torch.complex64, device="cuda"))
    assert empty.shape == (0, M, L // a)


def test_linearity_and_determinism(torch_cuda, nsdgt):
    torch = torch_cuda
    wl = CONFIGS[2]
    g = window(wl)
    f = batch(wl, 0, 3)
    plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype)
    ft = torch.from_numpy(f).cuda()
    c = plan.execute(ft)
    c2 = plan.execute(ft)
    assert torch.equal(c, c2)
    s = plan.execute((ft[0:1] + 2 * ft[1:2]).contiguous())
    assert rel((c[0] + 2 * c[1]).cpu().numpy(), s[0].cpu().numpy()) < 1e-5


def test_fast_path_matches_generic(torch_cuda, nsdgt):
    """Where a specialised kernel exists it agrees with the generic kernels (DGT_FORCE_GENERIC:
    the runtime-radix chunk kernels only): the fused kernel (configs 3, 5, kernel_path 2), the
    compile-time config-2 kernels, the config-4 front path (4) and the one-CTA path (config 1, 8)."""
    torch = torch_cuda
    for k, path in ((3, 2), (5, 2), (2, 0), (4, 4), (1, 8)):
        wl = CONFIGS[k - 1]
        g = window(wl)
        f = batch(wl, 0, min(wl.W, 2))
        pf = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype, real_input=wl.real_input)
        assert pf.info["kernel_path"] == path, (k, pf.info["kernel_path"])
        pg = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype, real_input=wl.real_input,
                        force_generic=True)
        assert pg.info["kernel_path"] == 0
        ft = torch.from_numpy(f).cuda()
        a_ = pf.execute(ft).cpu().numpy()
        b_ = pg.execute(ft).cpu().numpy()
        assert rel(a_, b_) <= TOL[wl.dtype]


def test_errors_on_gpu(torch_cuda, nsdgt):
    torch = torch_cuda
    with pytest.raises(nsdgt.DgtError) as ei:
        nsdgt.Plan(100, 8, 12, 1, 2, np.ones(100), dtype="c64")
    assert ei.value.status == 4 and ei.value.L_min == 48
    plan = nsdgt.Plan(48, 4, 6, 1, 2, np.ones(48), dtype="c64")
    with pytest.raises(TypeError):
        plan.execute(torch.zeros(48, dtype=torch.complex128, device="cuda"))


def test_binding_argument_checks(torch_cuda, nsdgt):
    """The ctypes binding validates what the C ABI cannot see (buffer lengths, dtypes, devices)
    before passing raw pointers: wrong window length, wrong host dtype / shape, bad outputs."""
    torch = torch_cuda
    L, a, M = 48, 4, 6
    with pytest.raises(ValueError):
        nsdgt.Plan(L, a, M, 1, 2, np.ones(L - 1), dtype="c64")   # would read past the window
    plan = nsdgt.Plan(L, a, M, 1, 2, np.ones(L), dtype="c128")
    f = np.random.default_rng(3).standard_normal((2, L)) + 0j
    ref = plan.execute(torch.from_numpy(f).cuda()).cpu().numpy()
    # numpy input is converted to the plan's dtype; torch input must match exactly
    assert np.array_equal(plan.execute_host(f), ref)
    assert np.allclose(plan.execute_host(f.astype(np.complex64)), ref, atol=1e-5)
    with pytest.raises(TypeError):
        plan.execute_host(torch.from_numpy(f.astype(np.complex64)))   # c64 data, c128 plan
    with pytest.raises(TypeError):
        plan.execute_host(torch.from_numpy(f).cuda())
    with pytest.raises(ValueError):
        plan.execute_host(np.zeros((2, L + 1), dtype=np.complex128))
    with pytest.raises(TypeError):
        plan.execute_host(f, out=np.zeros((2, M, L // a), dtype=np.complex64))
    with pytest.raises(TypeError):
        plan.execute(torch.from_numpy(f).cuda(), out=torch.zeros((1, M, L // a), dtype=torch.complex128, device="cuda"))


FIG2 = [(a, M, lam2) for a, M in [(32, 64), (40, 60), (60, 80)] for lam2 in (1, 2, 3, 5, 7, 10)]


@pytest.mark.parametrize("a,M,lam2", FIG2)
def test_fig2_grid_sampled(torch_cuda, nsdgt, oracle_mod, a, M, lam2):
    """The Fig. 2 lattices (L = lcm(a, M) 2520, lambda = 1/lambda2) that
    tools/fig2_sweep.py times: one signal, sampled columns against the oracle (c64)."""
    torch = torch_cuda
    L = a * M // math.gcd(a, M) * 2520
    lam1 = 0 if lam2 == 1 else 1
    g = pgauss_c(L, a * M / L)
    f, _ = random_pair(L, 60 + lam2, dtype="c64")
    plan = nsdgt.Plan(L, a, M, lam1, lam2, g, dtype="c64")
    c = plan.execute(torch.from_numpy(f).cuda())
    cols = np.sort(np.random.default_rng(lam2).choice(L // a, 12, replace=False))
    ref = oracle_mod.dgt(f, g, a, M, lam1, lam2, cols=cols)
    assert rel(c[:, torch.from_numpy(cols).cuda()].cpu().numpy(), ref) <= TOL["c64"], plan.info


def pgauss_c(L, tfr):
    from synthetic import pgauss
    return pgauss(L, tfr).astype(np.complex64)


@pytest.mark.parametrize("lam2", [1, 2])
def test_large_inner_length_global_scratch(torch_cuda, nsdgt, oracle_mod, lam2):
    """Fig. 2 lattice (60, 80) in complex128 with a time shear / separable: the inner Zak length
    d = 2520 needs 7 d 16 B of buffers per CTA, beyond shared memory, so the Zak kernels run on
    per-CTA global scratch.  Forward on sampled columns and synthesis of one signal."""
    torch = torch_cuda
    a, M = 60, 80
    L = a * M // math.gcd(a, M) * 2520
    lam1 = 0 if lam2 == 1 else 1
    f, g = random_pair(L, 70 + lam2, dtype="c128")
    plan = nsdgt.Plan(L, a, M, lam1, lam2, g, dtype="c128")
    assert plan.info["d"] == 2520
    c = plan.execute(torch.from_numpy(f).cuda())
    cols = np.sort(np.random.default_rng(lam2).choice(L // a, 8, replace=False))
    ref = oracle_mod.dgt(f, g, a, M, lam1, lam2, cols=cols)
    assert rel(c[:, torch.from_numpy(cols).cuda()].cpu().numpy(), ref) <= TOL["c128"]
    cr = np.random.default_rng(5).standard_normal((M, L // a)) + 0j
    fi = plan.inverse(torch.from_numpy(cr).cuda()).cpu().numpy()
    assert rel(fi, oracle_mod.idgt(cr, g, a, M, lam1, lam2)) <= TOL["c128"]


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_config2_compile_time_zak_matches_runtime(torch_cuda, nsdgt, oracle_mod, dtype, monkeypatch):
    """Config 2's lattice (d = 720, M' = 200): the compile-time Zak kernels (radix 9, 16, 5) and
    output DFT (radix 5, 8, 5) against the runtime-radix kernels, forward and synthesis, and
    against the oracle on sampled columns."""
    torch = torch_cuda
    wl = CONFIGS[1]
    g = window(wl)
    f = batch(wl, 0, 2).astype(np.complex64 if dtype == "c64" else np.complex128)
    ft = torch.from_numpy(f).cuda()
    pc = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=dtype)
    cc = pc.execute(ft)
    fc = pc.inverse(cc)
    monkeypatch.setenv("NSDGT_ZAK_RT", "1")
    monkeypatch.setenv("NSDGT_OUT_GENERIC", "1")
    pr = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=dtype)
    cr = pr.execute(ft)
    fr = pr.inverse(cr)
    assert rel(cc.cpu().numpy(), cr.cpu().numpy()) <= TOL[dtype]
    assert rel(fc.cpu().numpy(), fr.cpu().numpy()) <= TOL[dtype]
    cols = np.sort(np.random.default_rng(2).choice(wl.N, 16, replace=False))
    ref = oracle_mod.dgt(f, g, wl.a, wl.M, wl.lam1, wl.lam2, cols=cols)
    assert rel(cc[:, :, torch.from_numpy(cols).cuda()].cpu().numpy(), ref) <= TOL[dtype]


def test_two_plans_on_two_streams(torch_cuda, nsdgt):
    """Distinct plans are independent (include/nsdgt.h): a fused-path plan and a
    frequency-shear plan executing concurrently on two streams give the results of sequential
    runs, bit for bit."""
    torch = torch_cuda
    wl3, wl4 = CONFIGS[2], CONFIGS[3]
    p3 = nsdgt.Plan(wl3.L, wl3.a, wl3.M, wl3.lam1, wl3.lam2, window(wl3), dtype="c64")
    p4 = nsdgt.Plan(wl4.L, wl4.a, wl4.M, wl4.lam1, wl4.lam2, window(wl4), dtype="c128")
    f3 = torch.from_numpy(batch(wl3, 0, 32)).cuda()
    f4 = torch.from_numpy(batch(wl4, 0, 2)).cuda()
    ref3 = p3.execute(f3).clone()
    ref4 = p4.execute(f4).clone()
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    for _ in range(3):
        with torch.cuda.stream(s1):
            c3 = p3.execute(f3, stream=s1)
        with torch.cuda.stream(s2):
            c4 = p4.execute(f4, stream=s2)
    torch.cuda.synchronize()
    assert torch.equal(c3, ref3) and torch.equal(c4, ref4)


def random_lattices(n, seed=11):
    """Random feasible lattices with L <= 4096, both branches, p = 1 and p > 1."""
    from paper_1307_4569_b200 import nsdgt as nd
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        a = int(rng.integers(2, 65))
        M = int(rng.integers(2, 97))
        l2 = int(rng.integers(1, 6))
        l1 = 0 if l2 == 1 else int(rng.integers(1, l2))
        if math.gcd(l1, l2) != 1:
            continue
        lmin = l2 * (a * M // math.gcd(a, M))
        if lmin > 4096:
            continue
        k = int(rng.integers(1, 4096 // lmin + 1))
        L = lmin * k
        if L * (L // a) * M > 3_000_000:
            continue
        try:
            nd.lattice_plan(L, a, M, l1, l2)
        except nd.DgtError:
            continue
        out.append((L, a, M, l1, l2))
    return out


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_random_larger_lattices(torch_cuda, nsdgt, oracle_mod, dtype):
    """Random feasible lattices up to L = 4096: full comparison with the oracle."""
    torch = torch_cuda
    branches = set()
    for i, (L, a, M, l1, l2) in enumerate(random_lattices(30, seed=11 if dtype == "c128" else 12)):
        f, g = random_pair(L, 400 + i, dtype=dtype)
        c, plan = run_gpu(nsdgt, torch, f, g, L, a, M, l1, l2, dtype)
        branches.add(plan.info["branch"])
        ref = oracle_mod.dgt(f, g, a, M, l1, l2)
        assert rel(c, ref) <= TOL[dtype], (L, a, M, l1, l2, plan.info)
    assert len(branches) >= 2


def random_midsize_lattices(n, seed):
    """Random feasible lattices with 4096 < L <= 2^18 (a, M up to 256, lambda2 up to 7)."""
    from paper_1307_4569_b200 import nsdgt as nd
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        a = int(rng.integers(2, 257))
        M = int(rng.integers(2, 257))
        l2 = int(rng.integers(1, 8))
        l1 = 0 if l2 == 1 else int(rng.integers(1, l2))
        if math.gcd(l1, l2) != 1 or a >= M * 4:
            continue
        lmin = l2 * (a * M // math.gcd(a, M))
        if lmin > (1 << 18):
            continue
        ks = [k for k in range(1, (1 << 18) // lmin + 1) if lmin * k > 4096]
        if not ks:
            continue
        L = lmin * int(rng.choice(ks))
        try:
            nd.lattice_plan(L, a, M, l1, l2)
        except nd.DgtError:
            continue
        out.append((L, a, M, l1, l2))
    return out


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_random_midsize_lattices_sampled(torch_cuda, nsdgt, oracle_mod, dtype):
    """Random feasible lattices with L up to 2^18 (beyond the full-comparison sweep): two
    signals per lattice, 8 sampled columns against the oracle, both shear branches."""
    torch = torch_cuda
    branches = set()
    for i, (L, a, M, l1, l2) in enumerate(random_midsize_lattices(14, seed=21 if dtype == "c128" else 22)):
        f1, g = random_pair(L, 700 + i, dtype=dtype)
        f2, _ = random_pair(L, 800 + i, dtype=dtype)
        f = np.stack([f1, f2])
        c, plan = run_gpu(nsdgt, torch, f, g, L, a, M, l1, l2, dtype)
        branches.add(plan.info["branch"])
        cols = np.sort(np.random.default_rng(i).choice(L // a, min(8, L // a), replace=False))
        ref = oracle_mod.dgt(f, g, a, M, l1, l2, cols=cols)
        assert rel(c[:, :, cols], ref) <= TOL[dtype], (L, a, M, l1, l2, plan.info)
    assert len(branches) >= 2


def test_full_size_covariances(torch_cuda, nsdgt):
    """SURVEY §4 T4 at config 5's full size on the fused path (no oracle): modulation by k
    channels rolls c along m; translation by x = a lambda2 j samples rolls c along n by
    lambda2 j with the phase exp(-2 pi i x (m + w(n)) / M)."""
    torch = torch_cuda
    wl = CONFIGS[4]
    g = window(wl)
    plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype="c64")
    f = batch(wl, 0, 1)[0].astype(np.complex128)
    l = np.arange(wl.L)
    k, j = 5, 3
    b = wl.L // wl.M
    x = wl.a * wl.lam2 * j
    fs = np.stack([f, f * np.exp(2j * np.pi * b * k * l / wl.L), np.roll(f, x)]).astype(np.complex64)
    c = plan.execute(torch.from_numpy(fs).cuda()).cpu().numpy().astype(np.complex128)
    assert rel(c[1], np.roll(c[0], k, axis=0)) <= 5e-5
    m = np.arange(wl.M)[:, None]
    n = np.arange(wl.N)[None, :]
    wn = ((n * wl.lam1) % wl.lam2) / wl.lam2
    ph = np.exp(-2j * np.pi * x * (m + wn) / wl.M)
    assert rel(c[2], ph * np.roll(c[0], wl.lam2 * j, axis=1)) <= 5e-5


def test_config4_cluster_output_variant(torch_cuda, nsdgt, monkeypatch):
    """The experiment variant of config 4's output kernel (NSDGT_OUTCL=1: clusters of 3 CTAs
    staging each output row in distributed shared memory, then contiguous stores) writes the
    same coefficients bit for bit (same arithmetic, other store order)."""
    torch = torch_cuda
    wl = CONFIGS[3]
    g = window(wl)
    f = torch.from_numpy(batch(wl, 0, 2)).cuda()
    c0 = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype="c128").execute(f)
    monkeypatch.setenv("NSDGT_OUTCL", "1")
    c1 = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype="c128").execute(f)
    assert torch.equal(c0, c1)


def test_factorised_chirp_matches_table(torch_cuda, nsdgt, monkeypatch):
    """zak_ct multiplies the load chirp as P(x0) W_d^{-sigD x0 s} R(s) (a d-entry table and an
    index shift of the Zak DFT's output, ZakArgs::chR) instead of the length-L table
    (NSDGT_CHR_OFF): config 2's lattice and config 4's lattice on the zak_ct path agree."""
    torch = torch_cuda
    for k in (2, 4):
        wl = CONFIGS[k - 1]
        g = window(wl)
        f = torch.from_numpy(batch(wl, 0, 1)).cuda()
        if k == 4:
            monkeypatch.setenv("NSDGT_FRONT_CUFFT", "1")
            monkeypatch.setenv("NSDGT_ZAK_CT", "1")
        c1 = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype="c128").execute(f)
        monkeypatch.setenv("NSDGT_CHR_OFF", "1")
        c0 = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype="c128").execute(f)
        monkeypatch.delenv("NSDGT_CHR_OFF")
        assert rel(c1.cpu().numpy(), c0.cpu().numpy()) <= 1e-12, k
