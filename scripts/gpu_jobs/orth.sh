# orthogonalisation kernels: solver parity tests, then the bench line (v2 vs LT_ORTH_V1=1)
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/orth_bench.json 2> gpurun_out/orth_bench.err
python -c "
import json;d=json.load(open('gpurun_out/orth_bench.json'));print('v2', round(d['value']), round(d['e2e']['value']), d['kernel_breakdown']['fgmres_orth'])"
LT_ORTH_V1=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/orth_bench1.json 2> gpurun_out/orth_bench1.err
python -c "
import json;d=json.load(open('gpurun_out/orth_bench1.json'));print('v1', round(d['value']), round(d['e2e']['value']), d['kernel_breakdown']['fgmres_orth'])"
