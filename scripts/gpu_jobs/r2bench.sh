# GPU boundary tests + the bench line of one config (no ncu)
TAG=${1:-r2}; CFG=${2:-4}; STEPS=${3:-3}
timeout 900 python -m pytest tests/test_gpu_boundary.py -q > gpurun_out/${TAG}_bnd.log 2>&1; tail -2 gpurun_out/${TAG}_bnd.log
timeout 1200 python bench.py --config $CFG --steps $STEPS > gpurun_out/${TAG}_bench_c${CFG}.json 2> gpurun_out/${TAG}_bench_c${CFG}.err; tail -3 gpurun_out/${TAG}_bench_c${CFG}.err
python -c "
import json;d=json.load(open('gpurun_out/${TAG}_bench_c${CFG}.json'))
print('value', d['value'], 'e2e', d['e2e']['value'], 'ms/step', d['ms_per_step'], 'prof ms/step', d['profiled_pass_ms_per_step'], 'launches', d['gpu_launches'])
print('roofline', d['roofline']); print('hbm', d['roofline_hbm']); print('agg', d['hbm_aggregate']); print('clocks', d['clocks'])
print('cpu', d['cpu_baseline']); print('hostcopy', d.get('jacobian_host_copy'))
for k,v in list(d['class_breakdown'].items())[:12]: print(' ', k, v)
for k,v in list(d['kernel_breakdown'].items())[:16]: print('   ', k, v)
"
