for gs in 16 37 8; do
  export NSDGT_GS=$gs
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); print('GS=$gs cfg5 %.3f ms'%d['ms_per_step'])"
  NSDGT_NOPERSIST=1 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); print('GS=$gs nopersist cfg5 %.3f ms'%d['ms_per_step'])"
done
unset NSDGT_GS
python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null
python -c "import json; d=json.load(open('/tmp/b.json')); print('cfg3 %.3f ms'%d['ms_per_step'])"
