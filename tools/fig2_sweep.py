"""Fig. 2 grid on B200: the forward DGT by the shear algorithm and by the
multiwindow algorithm (dgt_plan_multiwindow) for lattice complexities lambda = 1/lambda2,
lambda2 = 1..10, at L = lcm(a, M) * 2520 for (a, M) in {(32, 64), (40, 60),
(60, 80)}; synthetic CN(0,1) signals, Gaussian window (tfr = a M / L), W signals per step.
Prints one JSON line per (lattice, algorithm): ms per step, coefficients/s, branch, shear,
kernel path.  The paper predicts the shear cost flat in lambda2 and the multiwindow cost
linear in it.
usage: python tools/fig2_sweep.py [W] [dtype] > profiles/r02_fig2_sweep.jsonl"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1307_4569_b200 as nsdgt
from synthetic import pgauss

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dtype = sys.argv[2] if len(sys.argv) > 2 else "c64"
cdt = torch.complex64 if dtype == "c64" else torch.complex128
for a, M in [(32, 64), (40, 60), (60, 80)]:
    L = a * M // math.gcd(a, M) * 2520
    g = pgauss(L, a * M / L)
    gen = torch.Generator(device="cuda").manual_seed(L)
    f = (torch.randn(W, L, dtype=cdt, device="cuda", generator=gen))
    for lam2, alg in [(l2, al) for l2 in range(1, 11) for al in ("shear", "multiwindow")]:
        lam1 = 0 if lam2 == 1 else 1
        try:
            plan = nsdgt.Plan(L, a, M, lam1, lam2, g, dtype=dtype, algorithm=alg)
        except nsdgt.DgtError as e:   # e.g. c128 inner Zak length beyond shared memory
            print(json.dumps({"a": a, "M": M, "L": L, "lambda": [lam1, lam2], "W": W, "dtype": dtype,
                              "algorithm": alg, "unsupported": str(e)}), flush=True)
            continue
        c = plan.execute(f)
        for _ in range(2):
            plan.execute(f, out=c)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        steps = 10
        for _ in range(steps):
            plan.execute(f, out=c)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        i = plan.info
        print(json.dumps({"a": a, "M": M, "L": L, "lambda": [lam1, lam2], "W": W, "dtype": dtype, "algorithm": alg,
                          "ms_per_step": ms,
                          "coefs_per_s": W * M * (L // a) / (ms * 1e-3), "branch": nsdgt.BRANCH_NAMES[i["branch"]],
                          "shear": [i["s0"], i["s1"]], "inner": [i["iM"], i["d"], i["p"], i["q"]],
                          "kernel_path": i["kernel_path"]}), flush=True)
        del plan, c
