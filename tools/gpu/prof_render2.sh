#!/bin/bash
# GPU box: ncu --set full of one forward and one backward render launch of the C2 bench step.
#   tools/gpu/prof_render2.sh TAG [extra env]
TAG=$1
python -c "import __graft_entry__ as g; g.build()" || exit 1
B="python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --breakdown-steps 1"
ncu --set full --clock-control none --import-source on -k regex:'k_render_bwd|k_render_fwd' \
    -s 6 -c 2 -o gpurun_out/prof_${TAG}_render $B > gpurun_out/prof_${TAG}_render.log 2>&1
tail -2 gpurun_out/prof_${TAG}_render.log
