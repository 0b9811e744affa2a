"""Quick check of the fused7 path: parity vs the oracle (sampled columns) and vs the v6 kernel, plus timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, paper_1307_4569_b200 as nsdgt
from synthetic import config, batch, window

def rel(x, y): return float(np.linalg.norm(x - y) / np.linalg.norm(y))

def timeit(p, f, c, reps=5):
    for _ in range(2): p.execute(f, out=c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): p.execute(f, out=c)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

for k, Wt in [(3, 256), (5, 1024)]:
    wl = config(k)
    g = window(wl)
    W = 5
    f = batch(wl, 0, W)
    ft = torch.from_numpy(f).cuda()
    p7 = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype)
    p6 = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype, force_generic=True)   # "v6" = generic reference
    print(f"cfg{k}: fused7 kernel_path={p7.info['kernel_path']} generic kernel_path={p6.info['kernel_path']}", flush=True)
    c7 = p7.execute(ft).cpu().numpy()
    c6 = p6.execute(ft).cpu().numpy()
    print(f"  rel(v7, v6) = {rel(c7, c6):.3e}", flush=True)
    cols = np.arange(0, wl.N, 97)
    ref = oracle.dgt(f, g, wl.a, wl.M, wl.lam1, wl.lam2, cols=cols)
    print(f"  rel(v7, oracle) = {rel(c7[:, :, cols], ref):.3e}   rel(v6, oracle) = {rel(c6[:, :, cols], ref):.3e}", flush=True)
    if rel(c7, c6) > 1e-4:
        d = np.abs(c7 - c6).max(axis=1)  # [W][N]
        bad = np.argwhere(d > 1e-3 * np.abs(c6).max())
        print("  first bad (w, n):", bad[:10].tolist(), flush=True)
    fb = torch.randn(Wt, wl.L, dtype=torch.complex64, device="cuda")
    cb = torch.empty(Wt, wl.M, wl.N, dtype=torch.complex64, device="cuda")
    t7 = timeit(p7, fb, cb); t6 = timeit(p6, fb, cb)
    gb = Wt * (wl.L * 8 + wl.M * wl.N * 8) / 1e9
    print(f"  W={Wt}: v7 {t7:.3f} ms ({gb / t7:.0f} GB/s)   v6 {t6:.3f} ms", flush=True)
