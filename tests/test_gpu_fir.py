"""Shear-OLA (dgt_plan_fir): the DGT with an FIR window computed block-wise must
equal Eq. (DGT) with the full-length window that is the FIR window zero-extended -- checked
against the oracle (sampled columns) and bit-for-bit-close against the full-length GPU plan."""
import numpy as np
import pytest

from synthetic import pgauss

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


def fir_window(Lg, dtype, seed):
    """A Gaussian-like FIR window of Lg taps in FIR order, with a random complex perturbation."""
    rng = np.random.default_rng(seed)
    t = np.concatenate([np.arange((Lg + 1) // 2), np.arange(-(Lg // 2), 0)])
    g = np.exp(-np.pi * (t / (Lg / 4)) ** 2) * (1 + 0.1 * (rng.standard_normal(Lg) + 1j * rng.standard_normal(Lg)))
    return g.astype(np.complex64 if dtype == "c64" else np.complex128)


def embed(g, L):
    Lg = len(g)
    out = np.zeros(L, dtype=g.dtype)
    t = np.concatenate([np.arange((Lg + 1) // 2), np.arange(-(Lg // 2), 0)])
    out[t % L] = g
    return out


CASES = [  # L, a, M, l1, l2, Lg, Lb, dtype
    (65536, 64, 256, 1, 2, 1024, 8192, "c64"),     # time shear (config 3's lattice)
    (65536, 64, 256, 1, 2, 777, 16384, "c128"),    # odd Lg
    (46080, 60, 240, 1, 3, 960, 5760, "c128"),     # frequency shear (config 4's lattice)
    (46080, 60, 240, 1, 3, 1201, 11520, "c64"),
    (24576, 32, 64, 0, 1, 300, 1536, "c64"),       # separable
    (36864, 48, 96, 2, 3, 500, 2304, "c128"),
]


@pytest.mark.parametrize("L,a,M,l1,l2,Lg,Lb,dtype", CASES)
def test_shear_ola_matches_full_length(torch_cuda, nsdgt, oracle_mod, L, a, M, l1, l2, Lg, Lb, dtype):
    torch = torch_cuda
    g = fir_window(Lg, dtype, L + Lg)
    rng = np.random.default_rng(L)
    W = 2
    f = (rng.standard_normal((W, L)) + 1j * rng.standard_normal((W, L))).astype(g.dtype)
    po = nsdgt.Plan(L, a, M, l1, l2, g, dtype=dtype, fir=True, Lb=Lb)
    assert po.info["kernel_path"] >= 16, po.info   # blocks, not the full-length fallback
    ft = torch.from_numpy(f).cuda()
    co = po.execute(ft).cpu().numpy()
    gL = embed(g, L)
    pf = nsdgt.Plan(L, a, M, l1, l2, gL, dtype=dtype)
    cf = pf.execute(ft).cpu().numpy()
    assert rel(co, cf) <= TOL[dtype]
    cols = np.sort(rng.choice(L // a, 16, replace=False))
    ref = oracle_mod.dgt(f, gL, a, M, l1, l2, cols=cols)
    assert rel(co[:, :, cols], ref) <= TOL[dtype]


def test_shear_ola_real_input_and_errors(torch_cuda, nsdgt, oracle_mod):
    """Real input, and the automatic block length: at L = 2^16 it would reach the whole signal,
    so the plan is the full-length plan of the zero-extended window (kernel path < 16)."""
    torch = torch_cuda
    L, a, M, l1, l2, Lg = 65536, 64, 256, 1, 2, 512
    g = fir_window(Lg, "c128", 3)
    f = np.random.default_rng(4).standard_normal((3, L))
    pa = nsdgt.Plan(L, a, M, l1, l2, g, dtype="c128", real_input=True, fir=True)
    assert pa.info["kernel_path"] < 16
    ca = pa.execute(torch.from_numpy(f).cuda()).cpu().numpy()
    po = nsdgt.Plan(L, a, M, l1, l2, g, dtype="c128", real_input=True, fir=True, Lb=4096)
    assert po.info["kernel_path"] >= 16
    co = po.execute(torch.from_numpy(f).cuda()).cpu().numpy()
    cols = np.arange(0, L // a, 97)
    assert rel(co[:, :, cols], oracle_mod.dgt(f, embed(g, L), a, M, l1, l2, cols=cols)) <= 1e-10
    assert rel(co, ca) <= 1e-10
    with pytest.raises(nsdgt.DgtError):
        nsdgt.Plan(L, a, M, l1, l2, g, dtype="c128", fir=True, Lb=1000)   # not a multiple of L_min
    with pytest.raises(nsdgt.DgtError):
        po.inverse(torch.zeros((1, M, L // a), dtype=torch.complex128, device="cuda"))
