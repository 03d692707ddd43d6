# ncu --set full of K4 and K6 (C4, one launch each), after a plain run of the same command
mkdir -p gpurun_out
CMD="python bench.py --config ${CONFIG:-C4} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k4_raster_fwd|k6_raster_bwd" -s 3 -c 2 \
    -o gpurun_out/prof_raster $CMD > gpurun_out/ncu_raster.log 2>&1
echo rc=$?
tail -1 gpurun_out/plain.log | cut -c1-200
