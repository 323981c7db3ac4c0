#!/bin/bash
# launch list (C2 bench + C4 driver), render + radix full captures with source
T=$1
python -c "import __graft_entry__ as g; g.build()" || exit 1
B="python bench.py --config C2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --breakdown-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${T}_C2.csv $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${T}_C4.csv python tools/prof_driver.py --config C4 --warmup 1 --steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_render_bwd|k_render_fwd' -s 6 -c 2 -o gpurun_out/prof_${T}_C2_render $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_radix|k_emit|k_key_ranges' -s 20 -c 8 -o gpurun_out/prof_${T}_C2_bin $B > /dev/null 2>&1
ls gpurun_out | grep $T
