#!/bin/bash
# GPU box: the round's evidence in one call -- the default bench line, the ncu launch list, the
# --set full captures (render, binning/projection, Adam) summarised ON THE BOX into small
# markdown/JSON files (the .ncu-rep files of binning and Adam are too large to bring back; the
# render capture is kept), the render SASS source pages and per-launch DRAM traffic.
#   tools/profile_round.sh TAG [CONFIG]
TAG=$1; CFG=${2:-C2}; OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
python bench.py --config $CFG > $OUT/${TAG}_bench_${CFG}.json 2> $OUT/${TAG}_bench_${CFG}.err
tools/profile.sh $TAG $CFG
mkdir -p $OUT/summ_$TAG
python tools/ncu_summary.py launches $OUT/launches_${TAG}_${CFG}.csv $OUT/summ_$TAG/${TAG}_${CFG}_launches.md > /dev/null
for K in render bin adam; do
  python tools/ncu_summary.py report $OUT/prof_${TAG}_${CFG}_$K.ncu-rep $OUT/summ_$TAG/${TAG}_${CFG}_$K.md > /dev/null
  python tools/ncu_summary.py traffic $OUT/prof_${TAG}_${CFG}_$K.ncu-rep $CFG $OUT/summ_$TAG/dram_traffic.json > /dev/null
done
for K in k_render_fwd k_render_bwd; do
  ncu -i $OUT/prof_${TAG}_${CFG}_render.ncu-rep -k regex:$K --page source --csv --print-source sass \
      > $OUT/summ_$TAG/sass_${TAG}_${K}.csv 2>/dev/null
done
rm -f $OUT/prof_${TAG}_${CFG}_bin.ncu-rep $OUT/prof_${TAG}_${CFG}_adam.ncu-rep $OUT/launches_${TAG}_${CFG}.log
du -sh $OUT
