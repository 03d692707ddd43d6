# A/B: BR_K4L_EKEEP (winner edge values kept for shading), C4 + C3 twice, then the parity tests
mkdir -p gpurun_out
for r in 1 2; do
VARIANTS="variants/lib_ek0.so variants/lib_ek1.so" CONFIGS="C4 C3" bash tools/ab_variants.sh
done > gpurun_out/ab_ekeep.txt 2>&1
cat gpurun_out/ab_ekeep.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3 > gpurun_out/ab_ekeep_parity.log
cat gpurun_out/ab_ekeep_parity.log
