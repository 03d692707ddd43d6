# C4 step time against a forced chunk length (--max-chunk; 0 = the automatic rule)
for g in ${GS:-0 1 2 3 4 6 8}; do
  timeout 600 python bench.py --config ${CFG:-C4} --max-chunk $g --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('G=$g', round(d['ms_per_step'],3), 'fwd', round(r['fwd_raster_ms'],3), 'bwd', round(r['bwd_raster_ms'],3))"
done
