# one compute-sanitizer tool per gpurun call (B200_PROFILING.md): TOOL=memcheck|racecheck|synccheck|initcheck
mkdir -p gpurun_out
python tools/sanitize_small.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool ${TOOL:-memcheck} --print-limit 50 python tools/sanitize_small.py \
    > gpurun_out/sanitize_${TOOL:-memcheck}.log 2>&1
echo "exit $?" >> gpurun_out/sanitize_${TOOL:-memcheck}.log
tail -5 gpurun_out/sanitize_${TOOL:-memcheck}.log
