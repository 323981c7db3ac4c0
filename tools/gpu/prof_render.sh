#!/bin/bash
# full-section captures of the render kernels in the C2 bench command (with source)
T=$1; CFG=${2:-C2}
python -c "import __graft_entry__ as g; g.build()" || exit 1
B="python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --breakdown-steps 1"
ncu --set full --clock-control none --import-source on -k regex:'k_render_bwd|k_render_fwd' -s 6 -c 2 -o gpurun_out/prof_${T}_${CFG}_render $B > /dev/null 2>&1
ls gpurun_out | grep $T
