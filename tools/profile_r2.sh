# Round-2 profile artefacts (C4 default bench): ncu launch list of one timed step and one ncu --set full
# capture of the raster kernels of a warm-up step.  Everything lands in gpurun_out/.
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_r2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_C4.csv $CMD > gpurun_out/ncu_launch_r2.log 2>&1
echo launches=$?
CMD1="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD1 > gpurun_out/plain1_r2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k4_raster_fwd|k6_raster_bwd" -s 4 -c 2 \
    -o gpurun_out/prof_r2_c4 $CMD1 > gpurun_out/ncu_full_r2.log 2>&1
echo full=$?
