set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_it.log 2>&1; echo rc=$? >> gpurun_out/t_it.log
timeout 300 python bench.py --config 4 --steps 20 > gpurun_out/b4_f.json 2>/dev/null
echo done
