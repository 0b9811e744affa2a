set -x
CFG=5 ENVS="NSDGT_FUSED=7;NSDGT_DBG=1;NSDGT_DBG=4097;NSDGT_FUSED=7" timeout 300 python tools/v7env.py > gpurun_out/env5.log 2>&1
echo done
