# quick GPU check: parity tests (optionally -k filter) + C4 kernel-only bench lines with/without an env A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -15 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-C4}; do
  for ab in "" ${AB_ENV}; do
    env $ab timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c [$ab]', round(d['value'],1), d['unit'], 'ms/step', round(d['ms_per_step'],3), 'fwd', round(r['fwd_raster_ms'],3), 'bwd', round(r['bwd_raster_ms'],3), 'frac', round(r['frac'],4))"
  done
done
