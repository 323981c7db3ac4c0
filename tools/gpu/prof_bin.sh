#!/bin/bash
# GPU box: ncu --set full of one launch of each binning kernel of the C2 bench step.
#   tools/gpu/prof_bin.sh TAG
TAG=$1
python -c "import __graft_entry__ as g; g.build()" || exit 1
B="python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --breakdown-steps 1"
ncu --set full --clock-control none --import-source on \
    -k regex:'k_emit|k_radix_scatter|k_seg_ranges|k_radix_hist|k_tile_counts' -s 40 -c 8 \
    -o gpurun_out/prof_${TAG}_bin $B > gpurun_out/prof_${TAG}_bin.log 2>&1
tail -2 gpurun_out/prof_${TAG}_bin.log
