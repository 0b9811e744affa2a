# config-4 kernel variants: parity subset + bench per variant (tools only)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -k "fbranch_out4096 or (full_size and 4) or fast_path or sweep or real_input or every_valid or config4_lattice" 2>&1 | tail -3
for v in "A=1" "NSDGT_ZAK_RT=1" $EXTRA; do
  env $v python bench.py --config 4 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['ms_per_step'],3), round(d['roofline']['frac'],4), [(k['name'], round(k['ms']/k['launches']*1000,1)) for k in d['roofline']['kernels']])"
done
