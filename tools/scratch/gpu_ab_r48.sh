# A/B: BR_K4L_R48 (48-B stage records), C4 + C3 twice, then the parity tests
mkdir -p gpurun_out
for r in 1 2; do
VARIANTS="variants/lib_r0.so variants/lib_r1.so" CONFIGS="C4 C3" bash tools/ab_variants.sh
done > gpurun_out/ab_r48.txt 2>&1
cat gpurun_out/ab_r48.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_soft.py -x -q 2>&1 | tail -3 > gpurun_out/ab_r48_parity.log
cat gpurun_out/ab_r48_parity.log
