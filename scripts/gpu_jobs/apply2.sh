# two-item apply: solver parity tests, inner-solve timing (v2 vs LT_APPLY_NI1=1), bench line
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
timeout 300 python scripts/perf_inner.py 4 80 > gpurun_out/ap2.log 2>&1; head -6 gpurun_out/ap2.log
LT_APPLY_NI1=1 timeout 300 python scripts/perf_inner.py 4 80 > gpurun_out/ap1.log 2>&1; head -6 gpurun_out/ap1.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/ap2_bench.json 2> gpurun_out/ap2_bench.err
python -c "
import json;d=json.load(open('gpurun_out/ap2_bench.json'));print('bench', round(d['value']), round(d['e2e']['value']), d['kernel_breakdown']['cocg_apply'])"
