set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
timeout 300 python bench.py --config 1 --steps 20 --no-cpu-baseline > gpurun_out/b1.json 2>gpurun_out/b1.err
NSDGT_TINY=0 timeout 300 python bench.py --config 1 --steps 20 --no-cpu-baseline > gpurun_out/b1_old.json 2>>gpurun_out/b1.err
timeout 300 python bench.py --config 1 --steps 20 --inverse --no-cpu-baseline > gpurun_out/b1_inv.json 2>>gpurun_out/b1.err
echo done
