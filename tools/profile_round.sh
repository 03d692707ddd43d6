# Round artefacts: default bench (C4), C5 and soft-C4 bench lines, the ncu launch list of the default
# bench and one ncu --set full capture of the raster kernels.  Everything lands in gpurun_out/.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench_c4=$?
timeout 900 python bench.py --config C5 --steps 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench_c5=$?
timeout 900 python bench.py --delta 1e-4 --no-cpu-baseline > gpurun_out/bench_c4_soft.json 2> gpurun_out/bench_c4_soft.err; echo bench_soft=$?
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo launches=$?
CMD1="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD1 > gpurun_out/plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k4_raster_fwd|k6_raster_bwd" -s 3 -c 2 \
    -o gpurun_out/prof_c4 $CMD1 > gpurun_out/ncu_full.log 2>&1
echo full=$?
bash tools/ncu_soft.sh > gpurun_out/ncu_soft_driver.log 2>&1
echo soft_full=$?
for c in C1 C2; do
  timeout 600 python bench.py --config $c --graph --steps 50 --no-cpu-baseline > gpurun_out/bench_${c}_graph.json 2> gpurun_out/bench_${c}_graph.err; echo graph_$c=$?
done
