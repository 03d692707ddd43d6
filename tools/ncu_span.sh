# ncu --set full of the span raster kernels on C4 (one timed step): K4 (skip the census launch) and K6
mkdir -p gpurun_out
CMD="env BLURRAST_RASTER=span python bench.py --config ${CFG:-C4} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_span.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k4s_raster_fwd|k6s_raster_bwd' -s 2 -c 2 \
    -o gpurun_out/prof_span ${CMD} > gpurun_out/ncu_span.log 2>&1
tail -3 gpurun_out/ncu_span.log
