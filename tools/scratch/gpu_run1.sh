# parity tests of the raster path + kernel-only bench lines (IMPLS="span legacy" for an A/B)
mkdir -p gpurun_out
BLURRAST_RASTER=${PARITY_IMPL:-span} timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -25 > gpurun_out/pt_parity.log
for impl in ${IMPLS:-span}; do
  if [ $impl = legacy ]; then unset BLURRAST_RASTER; else export BLURRAST_RASTER=span; fi
  for c in ${CONFIGS:-C4 C3 C2}; do
    timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$impl $c', round(d['value'],1), d['unit'], 'ms/step', round(d['ms_per_step'],3), 'fwd', round(r['fwd_raster_ms'],3), 'bwd', round(r['bwd_raster_ms'],3), 'frac', round(r['frac'],4), 'exec', r['executed_pair_tests_per_launch'])" >> gpurun_out/ab1.log 2>&1
  done
done
