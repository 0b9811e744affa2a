import torch, numpy as np, json, sys
sys.path.insert(0, '.')
import paper_1307_4569_b200 as nsdgt
from synthetic import config, window, batch
wl = config(5)
plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, window(wl), dtype="c64")
f = torch.from_numpy(batch(wl, 0, 64)).cuda()
res = {}
for W in (1024, 512, 256, 128):
    fw = f.repeat((W + 63) // 64, 1)[:W].contiguous()
    c = torch.empty((W, wl.M, wl.N), dtype=torch.complex64, device="cuda")
    for _ in range(3): plan.execute(fw, out=c)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n): plan.execute(fw, out=c)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    res[W] = ms
    print(W, round(ms, 4), "ms", "per-signal us", round(ms * 1000 / W, 3), "eff vs 1024:", round((res[1024] / 1024) / (ms / W), 3))
    del c, fw
