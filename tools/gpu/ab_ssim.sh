#!/bin/bash
# A/B of the D-SSIM loss: tag:ENV=VAL pairs, C2 --loss ssim
P=$1; shift
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu_ssim.py -q -x 2>&1 | grep -E "^E |passed|failed" | head -5
for spec in "$@"; do
  IFS=: read tag ev <<< "$spec"
  timeout 600 env $ev python bench.py --config C2 --loss ssim --steps 5 --no-cpu-baseline --no-e2e \
      --json-out gpurun_out/${P}_$tag.json > gpurun_out/${P}_$tag.log 2>&1
  python -c "import json; d=json.load(open('gpurun_out/${P}_$tag.json')); print('$tag', d['value'], d['calls_ms'].get('loss'))" \
      || tail -5 gpurun_out/${P}_$tag.log
done
