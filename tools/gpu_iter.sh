set -x
timeout 900 python -m pytest tests/test_gpu_tiny.py -x -q > gpurun_out/t_tiny.log 2>&1; echo rc=$? >> gpurun_out/t_tiny.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t_it.log 2>&1; echo rc=$? >> gpurun_out/t_it.log
echo done
