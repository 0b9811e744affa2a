"""Per-source-line stall breakdown from an ncu source page CSV (--print-source cuda,sass)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
reasons = sys.argv[2].split(",") if len(sys.argv) > 2 else ["stall_long_sb", "stall_mio", "stall_lg", "stall_barrier", "stall_short_sb", "stall_wait", "stall_not_selected", "stall_selected", "stall_math"]
cur = None
hdr = None
agg = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "":
        continue
    d = dict(zip(hdr, r))
    key = (cur, r[0], r[1][:70])
    for rs in reasons:
        try:
            agg.setdefault(rs, []).append((int(d.get(rs, "0") or 0), key))
        except ValueError:
            pass
for rs in reasons:
    lst = sorted(agg.get(rs, []), reverse=True)[:6]
    tot = sum(x[0] for x in agg.get(rs, []))
    print(f"== {rs} total {tot}")
    for n, (f, ln, src) in lst:
        if n:
            print(f"   {n:>8} {f}:{ln} {src}")
