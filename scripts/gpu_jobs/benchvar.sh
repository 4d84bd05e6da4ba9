timeout 900 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prof  ', d['value'], d['e2e']['value'], d['ms_per_step'])"
LT_BENCH_NOPROF=1 timeout 900 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('noprof', d['value'], d['e2e']['value'], d['ms_per_step'])"
