"""Phase times of config 2's two kernels (tools only; run in a copy whose libnsdgt.so is the
-DNSDGT_KTRACE build, tools/altrun.sh): block (0, 0)'s %globaltimer at phase boundaries, L2
flushed before each step.  zak_ct<720>: 0 start, 1 gather done, 2 DFT_720, 3 products,
4 four DFT_720s, 5 scatter; out_kernel<200>: 10 start, 11 loads, 12 DFT_200, 13 stores."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1307_4569_b200 as nsdgt
from paper_1307_4569_b200 import nsdgt as _m
from synthetic import CONFIGS, batch, window

lib = _m._lib
wl = CONFIGS[1]
p = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, window(wl), dtype="c128")
f = torch.from_numpy(batch(wl, 0, 1)).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
buf = (ctypes.c_ulonglong * 64)()
rows = []
for it in range(15):
    flush.zero_()
    p.execute(f)
    torch.cuda.synchronize()
    lib.dgt_debug_ktrace(buf)
    t = [buf[i] for i in range(64)]
    rows.append({"zak_gather": t[1] - t[0], "zak_dft1": t[2] - t[1], "zak_products": t[3] - t[2], "zak_dft4": t[4] - t[3],
                 "zak_scatter": t[5] - t[4], "gap_zak_end_to_out_start": t[10] - t[5], "out_loads": t[11] - t[10],
                 "out_dft": t[12] - t[11], "out_stores": t[13] - t[12]})
med = {k: sorted(r[k] for r in rows)[len(rows) // 2] for k in rows[0]}
print(json.dumps(med))
