"""Shear-OLA vs the full-length shear algorithm for long signals with short FIR windows
(PAPER.md:815-831, 921-949).  One JSON line per case (tools only).
usage: python tools/ola_bench.py > profiles/r01_ola.jsonl"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1307_4569_b200 as nsdgt


def fir_window(Lg):
    t = np.concatenate([np.arange((Lg + 1) // 2), np.arange(-(Lg // 2), 0)])
    return np.exp(-np.pi * (t / (Lg / 4)) ** 2).astype(np.complex64)


def embed(g, L):
    Lg = len(g)
    out = np.zeros(L, dtype=g.dtype)
    t = np.concatenate([np.arange((Lg + 1) // 2), np.arange(-(Lg // 2), 0)])
    out[t % L] = g
    return out


def timeit(plan, f, c, steps=5):
    plan.execute(f, out=c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        plan.execute(f, out=c)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


for (L, a, M, l1, l2, Lg, W) in [(1 << 22, 64, 256, 1, 2, 1024, 4), (1 << 22, 64, 256, 1, 2, 4096, 4),
                                 (737280 * 4, 60, 240, 1, 3, 960, 2), (1 << 22, 128, 512, 1, 2, 2048, 4)]:
    g = fir_window(Lg)
    f = torch.randn(W, L, dtype=torch.complex64, device="cuda")
    c = torch.empty(W, M, L // a, dtype=torch.complex64, device="cuda")
    pf = nsdgt.Plan(L, a, M, l1, l2, embed(g, L), dtype="c64")
    t_full = timeit(pf, f, c)
    c_full = c.clone()
    Lmin = nsdgt.lattice_plan(L, a, M, l1, l2)["L_min"]
    for Lb in (0, 1 << 16, 1 << 18):
        Lb = Lb if Lb == 0 else (Lb // Lmin) * Lmin
        if Lb and L % Lb:
            continue
        po = nsdgt.Plan(L, a, M, l1, l2, g, dtype="c64", fir=True, Lb=Lb)
        t_ola = timeit(po, f, c)
        err = float((c - c_full).norm() / c_full.norm())
        print(json.dumps({"L": L, "a": a, "M": M, "lambda": [l1, l2], "Lg": Lg, "W": W, "dtype": "c64",
                          "Lb": Lb or "auto", "ola_ms": t_ola, "full_ms": t_full, "full_over_ola": t_full / t_ola,
                          "ola_coefs_per_s": W * M * (L // a) / (t_ola * 1e-3), "ola_vs_full_rel_l2": err,
                          "ola_info": {k: po.info[k] for k in ("chunk", "kernel_path", "workspace_bytes")},
                          "full_inner": [pf.info[k] for k in ("branch", "d", "iM", "kernel_path")]}), flush=True)
        del po
    del pf, f, c, c_full
