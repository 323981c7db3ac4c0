#!/bin/bash
# A/B environment knobs on the bench workload (GPU box):
#   tools/ab_env.sh TAG CONFIG "GS_X=a GS_Y=b" "GS_X=c" ...
# Each variant runs bench.py (5 timed steps) and prints views/s, the render call times and
# their roofline fractions; JSON lines land in gpurun_out/ab_TAG_<i>.json.
TAG=$1; CFG=$2; shift 2
python -c "import __graft_entry__ as g; g.build()" || exit 1
i=0
for V in "$@"; do
  env $V python bench.py --config $CFG --steps 5 --warmup 3 --no-e2e --no-cpu-baseline \
      --json-out gpurun_out/ab_${TAG}_$i.json > /dev/null 2> gpurun_out/ab_${TAG}_$i.err
  python - "$V" gpurun_out/ab_${TAG}_$i.json <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[2]))
    print("%-40s %8.2f views/s" % (sys.argv[1], d["value"]),
          {k: d["calls_ms"][k] for k in ("render_fwd", "render_bwd", "bin_sort", "adam") if k in d["calls_ms"]},
          {k: d["rooflines"][k]["frac"] for k in ("render_fwd", "render_bwd")})
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
  i=$((i+1))
done
