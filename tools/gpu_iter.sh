timeout 300 ./tools/loadbench > gpurun_out/loadbench2.log 2>&1
echo done
