#!/bin/bash
# One GPU call: the bench line, then (after it exited 0) the ncu launch list of the same
# command and --set full captures of the top kernels.  Outputs under gpurun_out/$TAG*.
# Usage (through scripts/gpu.sh): bash scripts/profile_round.sh TAG [KERNEL_REGEX:SKIP ...]
set -u
TAG=${1:-r1}
shift || true
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err || { echo "bench failed"; tail -20 $OUT/${TAG}_bench.err; exit 1; }
cat $OUT/${TAG}_bench.json
# launch list: skip the warm-up build, record one timed build (~12k launches)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 10000 -c 9500 --csv \
  --log-file $OUT/${TAG}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
  > $OUT/${TAG}_ncu_launch.log 2>&1 || echo "launch list failed"
for KS in "$@"; do   # kernel_regex:launches_to_skip
  K=${KS%%:*}; S=${KS##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" --launch-skip "$S" -c 1 \
    -o $OUT/${TAG}_full_$K -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
    > $OUT/${TAG}_ncu_full_$K.log 2>&1 || echo "full capture $K failed"
done
ls -la $OUT