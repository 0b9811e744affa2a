"""Extract key metrics + stall samples of the kernels in an .ncu-rep into JSON (tools only).
usage: python tools/ncu_keys.py REPORT.ncu-rep OUT.json"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
if sys.argv[1].endswith(".csv"):   # a raw page exported on the GPU box (ncu -i R --page raw --csv)
    out = open(sys.argv[1]).read()
else:
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
res = []
for row in rows[2:]:
    d = dict(zip(hdr, row))
    u = dict(zip(hdr, units))
    k = {"kernel": d.get("Kernel Name", "")}
    for key in KEYS:
        if key in d:
            k[key] = [d[key], u.get(key, "")]
    st = {}
    for key, v in d.items():
        if "pcsamp_warps_issue_stalled_" in key and not key.endswith("not_issued"):
            try:
                st[key.split("stalled_")[1]] = int(float(v))
            except ValueError:
                pass
    k["stall_samples"] = dict(sorted(st.items(), key=lambda kv: -kv[1])[:14])
    res.append(k)
json.dump(res, open(sys.argv[2], "w"), indent=1)
print(f"{len(res)} kernel(s) -> {sys.argv[2]}")
