set -x
CFG=5 ENVS="NSDGT_FUSED=7;NSDGT_FUSED=7" timeout 300 python tools/v7env.py > gpurun_out/env5.log 2>&1
for v in NOFR NOG ALL; do
CFG=5 ENVS="NSDGT_FUSED=7;NSDGT_DBG=4" timeout 300 bash tools/altlib_run.sh tools/libnsdgt_xp_$v.so > gpurun_out/env5_$v.log 2>&1
done
echo done
