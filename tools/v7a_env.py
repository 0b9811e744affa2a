"""Time the fused synthesis kernel under a list of environment settings (tools only):
ENVS='NSDGT_LAG_ADJ=1;NSDGT_LAG_ADJ=2' CFG=5 WT=1024 python tools/v7a_env.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1307_4569_b200 as nsdgt
from synthetic import config, window
k = int(os.environ.get("CFG", "5")); Wt = int(os.environ.get("WT", "1024"))
wl = config(k); g = window(wl)
cb = torch.randn(Wt, wl.M, wl.N, dtype=torch.complex64, device="cuda")
fb = torch.empty(Wt, wl.L, dtype=torch.complex64, device="cuda")
keys = set()
for spec in os.environ.get("ENVS", "A=1").split(";"):
    env = dict(kv.split("=") for kv in spec.split() if "=" in kv)
    for kk in keys: os.environ.pop(kk, None)
    keys |= set(env)
    os.environ.update(env)
    p = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype)
    for _ in range(2): p.inverse(cb, out=fb)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): p.inverse(cb, out=fb)
    e1.record(); torch.cuda.synchronize()
    print(f"cfg{k} W={Wt} [{spec}]: {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)
    del p
