# usage: bash tools/prof_cmd.sh <tag> <bench args...>
tag=$1; shift
python bench.py "$@" --no-e2e --no-cpu-baseline > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o gpurun_out/prof_$tag python bench.py "$@" --no-e2e --no-cpu-baseline > gpurun_out/ncu_$tag.log 2>&1
echo rc=$?
