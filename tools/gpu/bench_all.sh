python -c "import __graft_entry__ as g; g.build()" || exit 1
for C in C1 C3 C4; do timeout 900 python bench.py --config $C > gpurun_out/r1p_bench_$C.json 2> gpurun_out/r1p_bench_$C.err; done
timeout 900 python bench.py --config C2 --loss ssim > gpurun_out/r1p_bench_C2_ssim.json 2> gpurun_out/r1p_bench_C2_ssim.err
timeout 900 python bench.py --config C2 --densify > gpurun_out/r1p_bench_C2_densify.json 2> gpurun_out/r1p_bench_C2_densify.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r1p_bench_ref.json 2> gpurun_out/r1p_bench_ref.err
for f in gpurun_out/r1p_bench_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d.get('value'), d.get('calls_ms'))" 2>&1 | cut -c1-300; done
