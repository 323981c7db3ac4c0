#!/bin/bash
# bench C2 with the L1 + D-SSIM loss, and a full ncu capture of the loss kernel
T=$1
python -c "import __graft_entry__ as g; g.build()" || exit 1
python bench.py --config C2 --loss ssim --steps 5 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_${T}_C2_ssim.json > gpurun_out/bench_${T}_C2_ssim.log 2>&1
python -c "import json; d=json.load(open('gpurun_out/bench_${T}_C2_ssim.json')); print(d['value'], d['calls_ms'], d['rooflines'].get('loss'))"
B="python bench.py --config C2 --loss ssim --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --breakdown-steps 1"
ncu --set full --clock-control none --import-source on -k regex:'k_ssim' -s 6 -c 2 -o gpurun_out/prof_${T}_C2_loss $B > /dev/null 2>&1
ls gpurun_out | grep $T
