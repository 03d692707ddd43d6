set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_soft.py -x -q -s 2>&1 | tail -25
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in C4 C3 C2; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --delta 1e-4 2>&1 | tail -1 > gpurun_out/soft_$c.json
  python -c "import json; d=json.load(open('gpurun_out/soft_$c.json')); r=d['roofline']; print('$c soft', round(d['value'],1), 'ms/step', round(d['ms_per_step'],3), 'fwd', round(r['fwd_raster_ms'],3), 'bwd', round(r['bwd_raster_ms'],3), 'softf', round(r['soft_fwd_ms'],3), 'softb', round(r['soft_bwd_ms'],3))"
done
