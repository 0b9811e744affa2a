import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1307_4569_b200 as nsdgt
from synthetic import config, window
k = int(os.environ.get("CFG", "5")); Wt = int(os.environ.get("WT", "1024"))
wl = config(k); g = window(wl)
fb = torch.randn(Wt, wl.L, dtype=torch.complex64, device="cuda")
cb = torch.empty(Wt, wl.M, wl.N, dtype=torch.complex64, device="cuda")
for dbg in [int(x) for x in os.environ.get("DBGS", "0,1,2,4,8,3,6,7,14,15").split(",")]:
    os.environ["NSDGT_DBG"] = str(dbg)   # read at plan time
    p = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype)
    for _ in range(2): p.execute(fb, out=cb)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): p.execute(fb, out=cb)
    e1.record(); torch.cuda.synchronize()
    print(f"cfg{k} W={Wt} dbg={dbg:2d}: {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)
    del p
