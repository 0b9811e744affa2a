"""Config-4 chunk-size sweep (tools only): ms per step of plan.execute over W = 16 for max_chunk
in {0 (auto), 1, 2, 4, 8}, events around the whole step (no per-kernel events)."""
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
for mc in (0, 1, 2, 4, 8):
    p = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype, max_chunk=mc)
    for _ in range(3):
        p.execute(f, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        p.execute(f, out=out)
    e1.record()
    e1.synchronize()
    res[f"chunk{mc}"] = e0.elapsed_time(e1) / 20
    del p
print(json.dumps(res))
