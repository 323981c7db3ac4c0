#!/bin/bash
# GPU-box helper: build, smoke, GPU tests, then bench lines for "tag:ENV=VAL:CONFIG" specs.
#   tools/gpu/ab_bench.sh PREFIX [--no-tests] C2:GS_X=1:C2 C2cull2:GS_RENDER_CULL=2:C2 ...
P=$1; shift
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
if [ "$1" == "--no-tests" ]; then shift; else
  timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "^E   |^FAILED|passed|failed" | cut -c1-300 | head -30
fi
for spec in "$@"; do
  IFS=: read tag ev cfg <<< "$spec"
  timeout 600 env $ev python bench.py --config $cfg --steps 5 --no-cpu-baseline --no-e2e \
      --json-out gpurun_out/${P}_$tag.json > gpurun_out/${P}_$tag.log 2>&1
  python -c "import json; d=json.load(open('gpurun_out/${P}_$tag.json')); print('$tag', d['value'], d['calls_ms'])" \
      || tail -5 gpurun_out/${P}_$tag.log
done
