set -x
timeout 900 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_multi_rank.py -x -q > gpurun_out/t_new.log 2>&1; echo rc=$? >> gpurun_out/t_new.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "full_size" > gpurun_out/t_par.log 2>&1; echo rc=$? >> gpurun_out/t_par.log
CFG=5 ENVS="NSDGT_FUSED=9;NSDGT_FUSED=7;NSDGT_FUSED=9;NSDGT_FUSED=7" timeout 300 python tools/v7env.py > gpurun_out/env5.log 2>&1
timeout 300 python bench.py --steps 10 > gpurun_out/bench_it.json 2> gpurun_out/bench_it.err
timeout 300 python bench.py --config 4 --steps 10 --no-cpu-baseline > gpurun_out/bench_it4.json 2> gpurun_out/bench_it4.err
echo done
