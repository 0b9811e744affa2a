"""Small-config latency experiment (tools only): configs 1-2, W = 1, L2 flushed before each step.
Times plan.execute on a stream with events, and the same execute captured in a CUDA graph."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1307_4569_b200 as nsdgt
from synthetic import CONFIGS, batch, window

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
res = {}
for k in (0, 1):
    wl = CONFIGS[k]
    g = window(wl)
    f = torch.from_numpy(batch(wl, 0, 1)).cuda()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        p = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype, real_input=wl.real_input, stream=st)
        out = torch.empty(1, wl.M, wl.N, dtype=torch.complex128, device="cuda")
        for _ in range(3):
            p.execute(f, out=out, stream=st)
        torch.cuda.synchronize()

        def timed(fn, n=30, fl=True):
            ts = []
            for _ in range(n):
                if fl:
                    flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                fn()
                e1.record(st)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            ts.sort()
            return ts[len(ts) // 2]

        res[f"cfg{k+1}_stream_flushed_us"] = timed(lambda: p.execute(f, out=out, stream=st))
        res[f"cfg{k+1}_stream_warm_us"] = timed(lambda: p.execute(f, out=out, stream=st), fl=False)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            p.execute(f, out=out, stream=st)
        torch.cuda.synchronize()
        res[f"cfg{k+1}_graph_flushed_us"] = timed(lambda: gr.replay())
        res[f"cfg{k+1}_graph_warm_us"] = timed(lambda: gr.replay(), fl=False)
        p.profile_begin()
        p.execute(f, out=out, stream=st)
        res[f"cfg{k+1}_kernels"] = [(s["name"], round(s["ms"] * 1e3, 2)) for s in p.profile_end()]
print(json.dumps(res))
