"""Time the fused cfg5/cfg3 kernel under the NSDGT_DBG knobs (which skip parts of the work)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1307_4569_b200 as nsdgt
from synthetic import config, window

def run(k, W, envs, reps=5):
    wl = config(k)
    g = window(wl)
    out = {}
    for tag, env in envs:
        for key in ("NSDGT_DBG", "NSDGT_NCOL", "NSDGT_GS", "NSDGT_DISCARD", "NSDGT_TMA", "NSDGT_PERSIST"):
            os.environ.pop(key, None)
        os.environ.update(env)
        p = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype)
        f = torch.randn(W, wl.L, dtype=torch.complex64, device="cuda")
        c = torch.empty(W, wl.M, wl.N, dtype=torch.complex64, device="cuda")
        for _ in range(3): p.execute(f, out=c)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps): p.execute(f, out=c)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out[tag] = ms
        print(f"cfg{k} W={W} {tag:28s} {ms:8.3f} ms", flush=True)
        del p, f, c
        torch.cuda.empty_cache()
    return out

envs = [("base", {}), ("ncol8", {"NSDGT_NCOL": "8"}), ("discard", {"NSDGT_DISCARD": "1"}),
        ("tma", {"NSDGT_TMA": "1"}), ("persist", {"NSDGT_PERSIST": "1"}),
        ("gs8", {"NSDGT_GS": "8"}), ("gs32", {"NSDGT_GS": "32"}), ("gs74", {"NSDGT_GS": "74"}),
        ("nofft(1)", {"NSDGT_DBG": "1"}), ("noMfft(2)", {"NSDGT_DBG": "2"}),
        ("noCstore(4)", {"NSDGT_DBG": "4"}), ("noOutStore(8)", {"NSDGT_DBG": "8"}),
        ("noAtile(16)", {"NSDGT_DBG": "16"}), ("noBtile(32)", {"NSDGT_DBG": "32"}),
        ("noProd(64)", {"NSDGT_DBG": "64"}), ("nofft+noMfft(3)", {"NSDGT_DBG": "3"}),
        ("allmem-off(60)", {"NSDGT_DBG": "60"}), ("fft-only(4+8+16+32+64=124)", {"NSDGT_DBG": "124"}),
        ("mem-only(1+2+64=67)", {"NSDGT_DBG": "67"})]
res = {"cfg5": run(5, 1024, envs), "cfg3": run(3, 256, envs[:8])}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/dbg_sweep.json", "w"), indent=1)
