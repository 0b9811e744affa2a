set -x
timeout 900 python -m pytest tests/test_gpu_multiwindow.py -x -q > gpurun_out/t_mw.log 2>&1; echo rc=$? >> gpurun_out/t_mw.log
timeout 600 python tools/fig2_sweep.py 8 c64 > gpurun_out/fig2_c64.jsonl 2> gpurun_out/fig2.err
timeout 600 python tools/fig2_sweep.py 4 c128 > gpurun_out/fig2_c128.jsonl 2>> gpurun_out/fig2.err
echo done
