# ncu --set full of the config-4 output kernel (tools only)
mkdir -p gpurun_out

ncu --set full --import-source on --clock-control none -k regex:"zak|out_f4096" -s 2 -c 2 -f -o gpurun_out/cfg4b \
  python bench.py --config 4 --steps 2 --warmup 3 > gpurun_out/ncu_cfg4b.log 2>&1
tail -3 gpurun_out/ncu_cfg4b.log
