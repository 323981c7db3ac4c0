python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_ssim.py -x -q 2>&1 | tail -1
for V in "" prev; do
  GS_LIB_VARIANT=$V python bench.py --loss ssim --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/ab_ssim_$V.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab_ssim_$V.json'));print('$V',d['value'],d['calls_ms']['loss'],d['rooflines']['loss']['frac'])"
done
