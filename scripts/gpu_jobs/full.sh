# GPU tests, smoke, bench line (no ncu)
TAG=${1:-r1v5}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gputests.log 2>&1; tail -3 gpurun_out/${TAG}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -2 gpurun_out/${TAG}_bench.err
python -c "
import json;d=json.load(open('gpurun_out/${TAG}_bench.json'))
print(d['value'], d['e2e']['value'], d['roofline'], d['clocks'], d['ms_per_step'])
for k,v in list(d['kernel_breakdown'].items())[:14]: print(k, v)
"
