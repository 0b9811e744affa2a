"""Relative l2 error of the CUDA path against the CPU oracle per BASELINE config (tools only):
every config at its full W in bench.py's launch configuration, signal 0 and the last signal
compared in full (all M x N coefficients) against the oracle (O1 literal for configs 1-2, O2
regrouped for 3-5, fp64, all host cores).  One JSON line per config.
usage: python tools/parity_report.py > profiles/r02_parity.jsonl"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_1307_4569_b200 as nsdgt
from synthetic import CONFIGS, batch, window

cores = len(os.sched_getaffinity(0))
for wl in CONFIGS:
    g = window(wl)
    f = batch(wl, 0, wl.W)
    plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype, real_input=wl.real_input)
    c = plan.execute(torch.from_numpy(f).cuda())
    torch.cuda.synchronize()
    variant = "literal" if wl.k <= 2 else "regrouped"
    errs, worst, secs = [], 0.0, 0.0
    num = den = 0.0
    for w in sorted({0, wl.W - 1}):
        t0 = time.perf_counter()
        ref = oracle.dgt(f[w], g, wl.a, wl.M, wl.lam1, wl.lam2, variant=variant, nthreads=cores)
        secs += time.perf_counter() - t0
        got = c[w].cpu().numpy()
        e = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
        worst = max(worst, e)
        num += float(np.linalg.norm(got - ref) ** 2)
        den += float(np.linalg.norm(ref) ** 2)
    tol = 1e-10 if wl.dtype == "c128" else 2e-5
    print(json.dumps({"config": wl.name, "dtype": wl.dtype, "W": wl.W, "signals_compared": sorted({0, wl.W - 1}),
                      "coefficients_compared": len({0, wl.W - 1}) * wl.M * wl.N, "rel_l2": (num / den) ** 0.5,
                      "worst_signal_rel_l2": worst, "tolerance": tol, "ok": worst <= tol,
                      "oracle": f"O{'1 literal' if variant == 'literal' else '2 regrouped'} fp64", "oracle_seconds": secs,
                      "cores": cores, "kernel_path": plan.info["kernel_path"]}), flush=True)
    del plan, c
