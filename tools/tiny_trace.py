"""Phase times of tiny_kernel (tools only; run in a copy whose libnsdgt.so is the -DNSDGT_TINY_TRACE build):
config 1, L2 flushed, block 0's %globaltimer at the phase boundaries."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1307_4569_b200 as nsdgt
from synthetic import CONFIGS, batch, window

from paper_1307_4569_b200 import nsdgt as _m
lib = _m._lib
wl = CONFIGS[0]
p = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, window(wl), dtype="c128", real_input=True)
f = torch.from_numpy(batch(wl, 0, 1)).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
buf = (ctypes.c_ulonglong * 16)()
rows = []
for it in range(10):
    flush.zero_()
    p.execute(f)
    torch.cuda.synchronize()
    lib.dgt_debug_tiny_trace(buf)
    t = [buf[i] for i in range(10)]
    rows.append([(t[i + 1] - t[i]) for i in range(9)])
names = ["loads", "dft_L", "gather", "dft_d1", "products", "dft_d2", "scatter", "dft_m", "output"]
med = [sorted(r[i] for r in rows)[len(rows) // 2] for i in range(9)]
print(json.dumps({"ns": dict(zip(names, med)), "total_ns": sum(med)}))
