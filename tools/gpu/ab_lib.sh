#!/bin/bash
# GPU box: bench the default libgs against in-tree A/B builds libgs_<name>.so (same box).
#   tools/gpu/ab_lib.sh CONFIG STEPS name1 name2 ...   (name "-" = the default build)
CFG=$1; STEPS=$2; shift 2
for V in "$@"; do
  if [ "$V" == "-" ]; then E=""; else E="GS_LIB_VARIANT=$V"; fi
  env $E python bench.py --config $CFG --steps $STEPS --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ab.out 2> /tmp/ab.err
  if ! tail -1 /tmp/ab.out | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['calls_ms']; print('%-6s %8.2f views/s fwd %.2f bwd %.2f bin %.2f adam %.2f proj %.2f' % ('$V', d['value'], c['render_fwd'], c['render_bwd'], c['bin_sort'], c['adam'], c['project']))" 2>/dev/null; then
    echo "$V FAILED:"; tail -5 /tmp/ab.err
  fi
done
