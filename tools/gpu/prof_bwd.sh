#!/bin/bash
# GPU box: ncu --set full of one render backward launch of the C2 bench step (library variant
# GS_LIB_VARIANT if set), summarised on the box.
#   tools/gpu/prof_bwd.sh TAG
TAG=$1
B="python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --breakdown-steps 1"
ncu --set full --clock-control none --import-source on -k regex:'k_render_bwd' -s 3 -c 1 \
    -o gpurun_out/prof_${TAG}_bwd $B > gpurun_out/prof_${TAG}_bwd.log 2>&1
python tools/ncu_summary.py report gpurun_out/prof_${TAG}_bwd.ncu-rep gpurun_out/prof_${TAG}_bwd.md > /dev/null
ncu -i gpurun_out/prof_${TAG}_bwd.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_${TAG}_bwd.csv 2>/dev/null
rm -f gpurun_out/prof_${TAG}_bwd.ncu-rep
tail -1 gpurun_out/prof_${TAG}_bwd.log
