timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "jacobian or predict" 2>&1 | tail -1
LT_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline 2> gpurun_out/trace.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])"
grep "\[lt\]   jacobian\|\[lt\]   expand" gpurun_out/trace.err | tail -4
