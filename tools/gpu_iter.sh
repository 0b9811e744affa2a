set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_it.log 2>&1; echo rc=$? >> gpurun_out/t_it.log
timeout 300 python bench.py --config 4 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/b4_f.json 2>/dev/null
NSDGT_FRONT_CUFFT=1 timeout 300 python bench.py --config 4 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/b4_rr.json 2>/dev/null
timeout 300 python tools/parity_report.py > gpurun_out/parity.jsonl 2>gpurun_out/parity.err
echo done
