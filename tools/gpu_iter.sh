set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_it.log 2>&1; echo rc=$? >> gpurun_out/t_it.log
timeout 300 python bench.py --config 4 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/b4_rr.json 2>/dev/null
NSDGT_ZAK_CT=1 timeout 300 python bench.py --config 4 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/b4_ct.json 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:zak --csv python bench.py --config 4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/l4.csv 2>/dev/null
echo done
