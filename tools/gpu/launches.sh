#!/bin/bash
# GPU box: ncu launch list (per-kernel device time, cold-cache, serialised) of one bench step.
#   tools/gpu/launches.sh TAG CONFIG
TAG=$1; CFG=${2:-C2}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_${CFG}.csv \
    python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --breakdown-steps 1 \
    > gpurun_out/launches_${TAG}_${CFG}.log 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_${TAG}_${CFG}.csv gpurun_out/launches_${TAG}_${CFG}.md > /dev/null
head -30 gpurun_out/launches_${TAG}_${CFG}.md
