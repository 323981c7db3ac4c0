#!/bin/bash
# Run on the GPU box (via gpurun): launch list + ncu --set full captures of the top kernels.
#   tools/profile.sh [tag] [config]
TAG=${1:-r1}
CFG=${2:-C2}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" || exit 1
B="python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --breakdown-steps 1"
# 1. every launch with its device time (cold-cache, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_${TAG}_${CFG}.csv $B \
    > $OUT/launches_${TAG}_${CFG}.log 2>&1
# 2. full sections of the render kernels and the fused backward+Adam kernel (4th step)
ncu --set full --clock-control none --import-source on -k regex:'k_render_bwd|k_render_fwd|k_bwd_adam' \
    -s 9 -c 3 -o $OUT/prof_${TAG}_${CFG}_main $B > $OUT/prof_${TAG}_${CFG}_main.log 2>&1
# 3. projection and binning kernels
ncu --set full --clock-control none --import-source on \
    -k regex:'k_project_count|k_project_write|k_rect_diff|k_place|k_sort_small' \
    -s 15 -c 5 -o $OUT/prof_${TAG}_${CFG}_bin $B > $OUT/prof_${TAG}_${CFG}_bin.log 2>&1
ls -la $OUT
