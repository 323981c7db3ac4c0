#!/bin/bash
# ncu --set full of the two render kernels on the bench workload + their SASS source pages.
#   tools/prof_render.sh TAG [CONFIG]
TAG=$1; CFG=${2:-C2}; OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
B="python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --breakdown-steps 1"
ncu --set full --clock-control none --import-source on -k regex:'k_render_bwd|k_render_fwd' \
    -s 6 -c 2 -o $OUT/prof_${TAG}_${CFG}_render $B > $OUT/prof_${TAG}_${CFG}_render.log 2>&1
for K in k_render_fwd k_render_bwd; do
  ncu -i $OUT/prof_${TAG}_${CFG}_render.ncu-rep -k regex:$K --page source --csv --print-source sass \
      > $OUT/sass_${TAG}_${K}.csv 2>/dev/null
done
ls -la $OUT | grep $TAG
