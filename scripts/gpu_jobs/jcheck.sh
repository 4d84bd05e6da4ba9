# Jacobian kernel change: parity tests touching the Jacobian, then the slice timing
TAG=${1:-jc}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "jacobian or predict" 2>&1 | tail -4
timeout 600 python scripts/perf_jac.py 128 2 > gpurun_out/${TAG}.log 2>&1
grep ' jacobian \| expand \|row0' gpurun_out/${TAG}.log
LT_JAC_MMA2=1 timeout 600 python scripts/perf_jac.py 128 2 > gpurun_out/${TAG}_mma2.log 2>&1
grep ' jacobian \|row0' gpurun_out/${TAG}_mma2.log
