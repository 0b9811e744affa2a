"""e2e (host buffers) vs raw PCIe copies for config 5 (tools only)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1307_4569_b200 as nsdgt
from synthetic import config, window
wl = config(5); g = window(wl); W = 1024
f_host = torch.randn(W, wl.L, dtype=torch.complex64).pin_memory()
c_host = torch.empty(W, wl.M, wl.N, dtype=torch.complex64, pin_memory=True)
p = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype="c64")
p.execute_host(f_host, out=c_host)
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); p.execute_host(f_host, out=c_host); torch.cuda.synchronize()
    print(f"execute_host: {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
dc = torch.empty(W, wl.M, wl.N, dtype=torch.complex64, device="cuda")
df = torch.empty(W, wl.L, dtype=torch.complex64, device="cuda")
torch.cuda.synchronize(); t = time.perf_counter(); c_host.copy_(dc); torch.cuda.synchronize()
print(f"raw D2H 8.6 GB: {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
torch.cuda.synchronize(); t = time.perf_counter(); df.copy_(f_host); torch.cuda.synchronize()
print(f"raw H2D 2.1 GB: {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t = time.perf_counter()
with torch.cuda.stream(s1): df.copy_(f_host, non_blocking=True)
with torch.cuda.stream(s2): c_host.copy_(dc, non_blocking=True)
torch.cuda.synchronize()
print(f"raw H2D || D2H: {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
