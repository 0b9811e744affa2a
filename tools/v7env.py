"""Time the fused7 kernel under a list of environment settings: ENVS='A=1 B=2;A=3' (semicolon-separated)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import threading, time, statistics
import torch
import paper_1307_4569_b200 as nsdgt
try:
    import pynvml
    pynvml.nvmlInit()
    _h = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:  # noqa: BLE001
    _h = None


def clock_sampler(stop, out):
    while not stop.is_set():
        try:
            out.append((pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(_h) / 1000,
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(_h)))
        except Exception:  # noqa: BLE001
            pass
        time.sleep(0.002)
from synthetic import config, window
k = int(os.environ.get("CFG", "5")); Wt = int(os.environ.get("WT", "1024"))
wl = config(k); g = window(wl)
fb = torch.randn(Wt, wl.L, dtype=torch.complex64, device="cuda")
cb = torch.empty(Wt, wl.M, wl.N, dtype=torch.complex64, device="cuda")
keys = set()
for spec in os.environ.get("ENVS", "").split(";"):
    env = dict(kv.split("=") for kv in spec.split() if "=" in kv)
    for kk in keys: os.environ.pop(kk, None)
    keys |= set(env)
    os.environ.update(env)
    p = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype)
    for _ in range(2): p.execute(fb, out=cb)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    samples, stop = [], threading.Event()
    th = threading.Thread(target=clock_sampler, args=(stop, samples)) if _h else None
    if th: th.start()
    e0.record()
    for _ in range(10): p.execute(fb, out=cb)
    e1.record(); torch.cuda.synchronize()
    if th: stop.set(); th.join()
    clk = statistics.median([x[0] for x in samples]) if samples else 0
    pw = max([x[1] for x in samples]) if samples else 0
    rs = 0
    for x in samples: rs |= x[2]
    print(f"cfg{k} W={Wt} [{spec.strip()}]: {e0.elapsed_time(e1) / 10:.3f} ms   sm {clk} MHz, max {pw:.0f} W, reasons 0x{rs:x}", flush=True)
    del p
