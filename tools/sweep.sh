python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null
python -c "import json; d=json.load(open('/tmp/b.json')); print('default cfg5 %.3f ms'%d['ms_per_step'])"
NSDGT_TMA=1 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null
python -c "import json; d=json.load(open('/tmp/b.json')); print('tma cfg5 %.3f ms'%d['ms_per_step'])"
python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null
python -c "import json; d=json.load(open('/tmp/b.json')); print('cfg3 %.3f ms'%d['ms_per_step'])"
