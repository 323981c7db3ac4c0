#!/bin/bash
# GPU box: bench lines of every config (C1, C3, C4; C2 with L1 + D-SSIM and with densification)
# and a short reference-arm (oracle) run, into gpurun_out/TAG_bench_*.json.
#   tools/gpu/bench_all.sh TAG
T=${1:-r1}
python -c "import __graft_entry__ as g; g.build()" || exit 1
for C in C1 C3 C4; do timeout 900 python bench.py --config $C > gpurun_out/${T}_bench_$C.json 2> gpurun_out/${T}_bench_$C.err; done
timeout 900 python bench.py --config C2 --loss ssim > gpurun_out/${T}_bench_C2_ssim.json 2> gpurun_out/${T}_bench_C2_ssim.err
timeout 900 python bench.py --config C2 --densify > gpurun_out/${T}_bench_C2_densify.json 2> gpurun_out/${T}_bench_C2_densify.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
for f in gpurun_out/${T}_bench_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d.get('value'), d.get('calls_ms'))" 2>&1 | cut -c1-300; done
