set -x
timeout 600 python -m pytest tests/test_gpu_inverse.py tests/test_gpu_fused7.py -x -q > gpurun_out/t_it.log 2>&1; echo rc=$? >> gpurun_out/t_it.log
timeout 300 python bench.py --inverse --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/inv5.json 2>/dev/null
timeout 300 python bench.py --config 3 --inverse --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/inv3.json 2>/dev/null
echo done
