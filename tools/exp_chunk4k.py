"""Config-4 per-kernel times at 1 and 16 signals per chunk (tools only): does the L2-resident
intermediate (47 MB per signal) make out_f4096 faster per signal?"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1307_4569_b200 as nsdgt
from synthetic import CONFIGS, batch, window

wl = CONFIGS[3]
g = window(wl)
f = torch.from_numpy(batch(wl, 0, wl.W)).cuda()
out = torch.empty(wl.W, wl.M, wl.N, dtype=torch.complex128, device="cuda")
res = {}
for mc in (1, 2, 16):
    p = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype, max_chunk=mc)
    for _ in range(3):
        p.execute(f, out=out)
    torch.cuda.synchronize()
    p.profile_begin()
    for _ in range(10):
        p.execute(f, out=out)
    st = p.profile_end()
    res[f"chunk{mc}"] = {k["name"]: round(k["ms"] / 10, 4) for k in st}
    del p
print(json.dumps(res))
