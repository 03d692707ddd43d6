# ncu --set full of chosen kernels in one C4 bench step (default: K4 and K6 of the default path)
# usage: KREGEX='k4_raster_fwd<0|k6_raster_bwd_fx' SKIP=2 COUNT=2 OUT=prof_x bash tools/ncu_kernels.sh
mkdir -p gpurun_out
CMD="python bench.py --config ${CFG:-C4} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_${OUT:-prof}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k4_raster_fwd<false, 0>|k6_raster_bwd_fx}" \
    -s ${SKIP:-2} -c ${COUNT:-2} -o gpurun_out/${OUT:-prof} ${CMD} > gpurun_out/ncu_${OUT:-prof}.log 2>&1
tail -2 gpurun_out/ncu_${OUT:-prof}.log
