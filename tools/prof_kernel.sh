# ncu --set full of kernels matching $KREGEX on config $CFG (one warm-up step) + per-line table
mkdir -p gpurun_out
CMD1="python bench.py --config ${CFG:-C4} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD1 > gpurun_out/plain1.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"$KREGEX" -s ${SKIP:-2} -c ${COUNT:-1} \
    -o gpurun_out/prof_${TAG:-x} $CMD1 > gpurun_out/ncu_full_${TAG:-x}.log 2>&1
python tools/ncu_lines2.py gpurun_out/prof_${TAG:-x}.ncu-rep "$KREGEX" 60 > gpurun_out/lines_${TAG:-x}.txt 2>&1
echo done
