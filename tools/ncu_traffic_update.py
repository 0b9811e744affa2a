"""Record per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the kernels in
an `ncu --set full` report into profiles/ncu_traffic.json under a workload name, keyed by the
profile-kind names bench.py reports (tools only).
usage: python tools/ncu_traffic_update.py REPORT.ncu-rep|RAW.csv WORKLOAD"""
import csv
import io
import json
import os
import subprocess
import sys

# CUDA kernel name prefix -> the profile kind of dgt.cu's prof_close (bench.py's kernel names)
KINDS = [("fused7a_kernel", "fused7a_t_p1"), ("fused7_kernel", "fused7_t_p1"),
         ("zak_ct_adj_kernel", "zak_adjoint"), ("zak_ct_kernel", "zak_ct"),
         ("zak_rr0_kernel", "zak_rr"), ("zak_rr_kernel", "zak_rr"), ("front_f4096_kernel", "front_f4096"),
         ("out_f4096_adj_kernel", "out_adjoint"), ("out_f4096_kernel", "out_f4096"),
         ("zak_adj_kernel", "zak_adjoint"), ("out_adj_kernel", "out_adjoint"),
         ("zak_kernel", "zak_generic"), ("out_kernel", "out_generic")]


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
    return float(v.replace(",", "")) * scale


def main():
    rep, workload = sys.argv[1], sys.argv[2]
    if rep.endswith(".csv"):   # a raw page exported on the GPU box
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    path = os.path.join(os.path.dirname(__file__), "..", "profiles", "ncu_traffic.json")
    table = json.load(open(path)) if os.path.exists(path) else {}
    entry = table.setdefault(workload, {})
    for row in rows[2:]:
        d = dict(zip(head, row))
        u = dict(zip(head, units))
        name = d.get("Kernel Name", "").removeprefix("void ")
        kind = next((k for p, k in KINDS if name.startswith(p)), None)
        if kind is None:
            continue
        t = sum(to_bytes(d[k], u[k]) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        entry[kind] = t
        print(workload, kind, t)
    json.dump(table, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
