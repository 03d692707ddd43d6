# Profile artefacts of the default C4 bench (tag $TAG, default r2d): ncu launch list of one timed step, and one
# ncu --set full capture of K4 (k4l_raster_fwd) and K6 (k6v_raster_bwd) of a warm-up step.  -> gpurun_out/
mkdir -p gpurun_out
TAG=${TAG:-r2d}
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches_C4.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo launches=$?
CMD1="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD1 > gpurun_out/plain1_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k4l_raster_fwd|k6v_raster_bwd" -s 2 -c 4 \
    -o gpurun_out/prof_${TAG}_c4 $CMD1 > gpurun_out/ncu_full_${TAG}.log 2>&1
echo full=$?
python tools/update_traffic.py gpurun_out/prof_${TAG}_c4.ncu-rep C4 'k4l_raster_fwd<0, 0>=k4l_raster_fwd' 'k6v_raster_bwd=k6v_raster_bwd'
python tools/ncu_stalls.py gpurun_out/prof_${TAG}_c4.ncu-rep k4l_raster k4l 14 > gpurun_out/${TAG}_stalls.txt 2>&1
python tools/ncu_stalls.py gpurun_out/prof_${TAG}_c4.ncu-rep k6v_raster k6v 14 >> gpurun_out/${TAG}_stalls.txt 2>&1
