#!/bin/bash
# A/B the render kernels' pixels-per-thread on the bench workload (GPU box).
CFG=${1:-C2}
python -c "import __graft_entry__ as g; g.build()" || exit 1
for P in 2 4 8; do
  GS_RENDER_PPT=$P python bench.py --config $CFG --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
      --json-out gpurun_out/ab_ppt${P}_${CFG}.json > /dev/null 2>&1
  python - <<PY
import json; d=json.load(open("gpurun_out/ab_ppt${P}_${CFG}.json"))
print("PPT=${P}", d["value"], {k: d["calls_ms"][k] for k in ("render_fwd","render_bwd")},
      {k: d["rooflines"][k]["frac"] for k in ("render_fwd","render_bwd")})
PY
done
