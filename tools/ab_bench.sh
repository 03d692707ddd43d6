# step / fwd / bwd ms of library variants (BLURRAST_LIB) on configs: VARIANTS="a b" CONFIGS="C4 C3"
for v in ${VARIANTS}; do for c in ${CONFIGS:-C4 C3}; do
  BLURRAST_LIB=$PWD/variants/lib_$v.so timeout 900 python bench.py --config $c $EXTRA --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v $c', round(d['ms_per_step'],3), 'fwd', round(r['fwd_raster_ms'],3), 'bwd', round(r['bwd_raster_ms'],3))" || echo "$v $c FAILED"
done; done
