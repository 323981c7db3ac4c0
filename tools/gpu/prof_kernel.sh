#!/bin/bash
# GPU box: ncu --set full of launches of the kernels matching REGEX in the C2 bench step.
#   tools/gpu/prof_kernel.sh TAG REGEX [SKIP] [COUNT] [CONFIG]
TAG=$1; RX=$2; SK=${3:-5}; CNT=${4:-1}; CFG=${5:-C2}
python -c "import __graft_entry__ as g; g.build()" || exit 1
B="python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --breakdown-steps 1"
ncu --set full --clock-control none --import-source on -k regex:"$RX" -s $SK -c $CNT \
    -o gpurun_out/prof_${TAG} $B > gpurun_out/prof_${TAG}.log 2>&1
tail -2 gpurun_out/prof_${TAG}.log
