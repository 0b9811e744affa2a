"""Phase trace of the fused7 kernel (NSDGT_DBG=16): per-CTA globaltimer stamps -> time per phase."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1307_4569_b200 as nsdgt
from synthetic import config, window
k = int(os.environ.get("CFG", "5")); Wt = int(os.environ.get("WT", "1024"))
wl = config(k); g = window(wl)
fb = torch.randn(Wt, wl.L, dtype=torch.complex64, device="cuda")
cb = torch.empty(Wt, wl.M, wl.N, dtype=torch.complex64, device="cuda")
os.environ["NSDGT_DBG"] = str(16 | int(os.environ.get("EXTRA", "0")))   # read at plan time
p = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, g, dtype=wl.dtype)
p.execute(fb, out=cb); torch.cuda.synchronize()
lib = nsdgt.nsdgt._lib
lib.dgt_debug_trace_log.restype = ctypes.c_void_p
lib.dgt_debug_trace_log.argtypes = [ctypes.c_void_p]
ptr = ctypes.c_uint64(lib.dgt_debug_trace_log(p._h) or 0)
cudart = ctypes.CDLL("libcudart.so") if os.path.exists("/usr/local/cuda/lib64/libcudart.so") else None
if cudart is None:
    import glob
    cudart = ctypes.CDLL(glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*"))[0])
buf = np.zeros(8 * 4096, dtype=np.uint64)
rc = cudart.cudaMemcpy(ctypes.c_void_p(buf.ctypes.data), ctypes.c_void_p(ptr.value), ctypes.c_size_t(buf.nbytes), 2)
assert rc == 0, rc
print("log ptr", hex(ptr.value), "nonzero entries", int((buf != 0).sum()), "lib", nsdgt.nsdgt.LIB_PATH if hasattr(nsdgt, "nsdgt") else "", flush=True)
names = {30: "A-prespin", 31: "B-prespin", 32: "B-prefetched", 1: "top", 2: "top(B)", 3: "after-bar1", 4: "after-spin", 5: "loaded", 6: "prefetched", 10: "tile-start",
         11: "stage1-done", 12: "xwritten", 13: "xbarrier", 14: "tile-end", 20: "fwd-done", 21: "F-barrier", 22: "gather-done"}
tot = {}
for c in range(8):
    e = buf[c * 4096:(c + 1) * 4096]
    e = e[e != 0]
    if len(e) < 2: continue
    t = (e >> 8).astype(np.int64); code = (e & 255).astype(np.int64)
    for i in range(1, len(e)):
        key = (names.get(int(code[i - 1]), code[i - 1]), names.get(int(code[i]), code[i]))
        tot[key] = tot.get(key, 0) + int(t[i] - t[i - 1])
    span = t[-1] - t[0]
total = sum(tot.values())
print(f"cfg{k} W={Wt}: {total / 1e6 / 8:.3f} ms per CTA traced (8 CTAs)")
for key, v in sorted(tot.items(), key=lambda x: -x[1])[:25]:
    print(f"  {100 * v / total:5.1f}%  {v / 8 / 1e3:9.1f} us/CTA   {key[0]:>12s} -> {key[1]}")
