# full GPU evidence run (gpurun): GPU tests, smoke, bench lines for every config (forward and
# synthesis), the reference arm, ncu launch lists and --set full captures, a functional
# two-rank run.  usage: bash tools/round_cmd.sh TAG   (outputs under gpurun_out/, *_TAG.*)
tag=$1
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_$tag.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_$tag.log
python __graft_entry__.py --smoke > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$tag.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks_$tag.csv &
SMI=$!
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
kill $SMI
for k in 1 2 3 4; do python bench.py --config $k --steps 20 --warmup 3 --cpu-budget 5 > gpurun_out/bench_cfg${k}_$tag.json 2>/dev/null; done
for k in 5 3 4 2 1; do python bench.py --config $k --inverse --steps 10 --warmup 3 --cpu-budget 5 > gpurun_out/bench_inv_cfg${k}_$tag.json 2>/dev/null; done
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$tag.json 2>/dev/null
python tools/parity_report.py > gpurun_out/parity_$tag.jsonl 2>/dev/null
NSDGT_DIST_BACKEND=gloo python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_n2_one_gpu_$tag.json 2>/dev/null
echo phase1 done
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_$tag.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu1_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused -s 1 -c 1 -o gpurun_out/prof_$tag python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu2_$tag.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4_$tag.csv python bench.py --config 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"zak|out_f4096|front" -s 3 -c 3 -o gpurun_out/prof_cfg4_$tag python bench.py --config 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused7 -s 1 -c 1 -o gpurun_out/prof_cfg3_$tag python bench.py --config 3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tiny -s 3 -c 1 -o gpurun_out/prof_cfg1_$tag python bench.py --config 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused7a -s 1 -c 1 -o gpurun_out/prof_inv_$tag python bench.py --inverse --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
# export the raw pages (small) and the source page of the config-5 capture; drop the reports
for r in gpurun_out/prof_*$tag.ncu-rep; do ncu -i $r --page raw --csv > ${r%.ncu-rep}_raw.csv 2>/dev/null; done
ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_${tag}_source.csv 2>/dev/null
rm -f gpurun_out/prof_*$tag.ncu-rep
du -sh gpurun_out
echo done
