# ncu --set full of the soft kernels (C3, one launch each of K8, K9C, K9), after a plain run of the same command
set -x
mkdir -p gpurun_out

CMD="python bench.py --config C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --delta 1e-4"
$CMD > gpurun_out/plain_soft.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k8_soft_fwd|k9c_soft_bwd|k9_soft_bwd" -s 3 -c 3 \
    -o gpurun_out/prof_soft $CMD > gpurun_out/ncu_soft.log 2>&1
echo rc=$?
tail -1 gpurun_out/plain_soft.log | cut -c1-300
