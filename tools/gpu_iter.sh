set -x
timeout 600 python -m pytest tests/test_gpu_fused7.py tests/test_gpu_inverse.py -x -q > gpurun_out/t_it.log 2>&1; echo rc=$? >> gpurun_out/t_it.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "full_size or fast_path or covariances" >> gpurun_out/t_it.log 2>&1; echo rc=$? >> gpurun_out/t_it.log
CFG=5 ENVS="NSDGT_FUSED=7;NSDGT_FUSED=7" timeout 300 python tools/v7env.py > gpurun_out/env5.log 2>&1
CFG=3 WT=256 ENVS="NSDGT_FUSED=7;NSDGT_FUSED=7" timeout 300 python tools/v7env.py > gpurun_out/env3.log 2>&1
echo done
