#!/bin/bash
# Run on the GPU box (via gpurun): launch list of the bench command + ncu --set full captures.
#   tools/profile.sh [tag] [config]
TAG=${1:-r1}
CFG=${2:-C2}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" || exit 1
B="python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --breakdown-steps 1"
# 1. every launch of the bench command with its device time (cold-cache, serialised: shares)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_${TAG}_${CFG}.csv $B \
    > $OUT/launches_${TAG}_${CFG}.log 2>&1
# 2. full sections of the render kernels in the bench command (4th step)
ncu --set full --clock-control none --import-source on -k regex:'k_render_bwd|k_render_fwd' \
    -s 6 -c 2 -o $OUT/prof_${TAG}_${CFG}_render $B > $OUT/prof_${TAG}_${CFG}_render.log 2>&1
# 3. projection and binning kernels in the bench command
ncu --set full --clock-control none --import-source on \
    -k regex:'k_project_count|k_project_write|k_radix_scatter|k_radix_hist|k_emit|k_fine|k_tile_counts|k_diff_rows|k_diff_cols' \
    -s 150 -c 20 -o $OUT/prof_${TAG}_${CFG}_bin $B > $OUT/prof_${TAG}_${CFG}_bin.log 2>&1
# 4. the Adam kernels write all parameters, moments and gradients (~11 GB at C2), which kernel
#    replay must save/restore: capture them on a reduced copy (4 views, 2.8M Gaussians)
D="python tools/prof_driver.py --config $CFG --views 4 --gaussians 2800000 --warmup 2 --steps 1"
ncu --set full --clock-control none --import-source on -k regex:'k_bwd_adam|k_adam_apply' \
    -s 4 -c 2 -o $OUT/prof_${TAG}_${CFG}_adam $D > $OUT/prof_${TAG}_${CFG}_adam.log 2>&1
ls -la $OUT | tail -5
