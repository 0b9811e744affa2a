"""Config-4 experiment (tools only): does splitting the step over two streams overlap the cuFFT
front end of one half with the zak_ct / out_f4096 kernels of the other?  Prints ms per step
for one plan over W = 16, chunk variants, and two plans of W / 2 on two streams."""
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
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, steps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        # join the side stream back into the current one before the end event
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


res = {}
p = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype)
out = torch.empty(wl.W, wl.M, wl.N, dtype=torch.complex128, device="cuda")
res["one_plan_W16"] = timeit(lambda: p.execute(f, out=out))
for mc in (2, 4, 8):
    q = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype, max_chunk=mc)
    res[f"one_plan_chunk{mc}"] = timeit(lambda: q.execute(f, out=out))
    del q
for parts in (2, 4):
    s = [torch.cuda.Stream() for _ in range(parts)]
    h = wl.W // parts
    plans = [nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype, stream=s[i]) for i in range(parts)]

    def two():
        cur = torch.cuda.current_stream()
        for i in range(parts):
            s[i].wait_stream(cur)
            plans[i].execute(f[i * h:(i + 1) * h], out=out[i * h:(i + 1) * h], stream=s[i])
        for i in range(parts):
            cur.wait_stream(s[i])

    res[f"{parts}_plans_{parts}_streams"] = timeit(two)

    def seq():
        cur = torch.cuda.current_stream()
        for i in range(parts):
            plans[i].execute(f[i * h:(i + 1) * h], out=out[i * h:(i + 1) * h], stream=cur)

    res[f"{parts}_plans_1_stream"] = timeit(seq)
    del plans
print(json.dumps(res))
