set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t_it.log 2>&1; echo rc=$? >> gpurun_out/t_it.log
for k in 2 4 5; do
timeout 300 python bench.py --config $k --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/b${k}_pdl.json 2>gpurun_out/b${k}.err
NSDGT_PDL_OFF=1 timeout 300 python bench.py --config $k --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/b${k}_nopdl.json 2>/dev/null
done
echo done
