# A/B of library variants built into variants/lib_*.so (kernel-only bench lines)
mkdir -p gpurun_out
for v in ${VARIANTS:-variants/lib_*.so}; do
  for c in ${CONFIGS:-C4 C3}; do
    BLURRAST_LIB=$PWD/$v timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline $EXTRA 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', '$c', round(d['ms_per_step'],3), 'fwd', round(r['fwd_raster_ms'],3), 'bwd', round(r['bwd_raster_ms'],3), r.get('kernels_ms',''))" || echo "$v $c FAILED"
  done
done
