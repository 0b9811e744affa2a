"""Summarise an ncu source page (CSV, --print-source cuda,sass) by CUDA source line."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur = None
hdr = None
out = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    d = dict(zip(hdr, r))
    try:
        samp = int(d["Warp Stall Sampling (All Samples)"])
        inst = int(d["Instructions Executed"])
    except (ValueError, KeyError):
        continue
    exc = d.get("L1 Wavefronts Shared Excessive", "0")
    exc = int(exc) if exc.isdigit() else 0
    out.append((samp, inst, exc, cur, r[0], r[1][:90]))
tot = sum(o[0] for o in out)
out.sort(reverse=True)
print("total samples", tot)
for o in out[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100*o[0]/tot:5.1f}%  inst={o[1]:>11}  smem_excess={o[2]:>10}  {o[3]}:{o[4]}  {o[5]}")
