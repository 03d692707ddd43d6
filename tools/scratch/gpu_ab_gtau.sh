# A/B: BR_K4L_GTAU (stage reads its taus from the global schedule, no S.taus write before the group barrier), C4 + C3 twice, C5 once,
# then the parity tests on the GTAU library
mkdir -p gpurun_out
for r in 1 2; do
VARIANTS="variants/lib_g0.so variants/lib_g1.so" CONFIGS="C4 C3" bash tools/ab_variants.sh
done > gpurun_out/ab_gtau.txt 2>&1
VARIANTS="variants/lib_g0.so variants/lib_g1.so" CONFIGS="C5" EXTRA="--steps 3 --warmup 3" bash tools/ab_variants.sh >> gpurun_out/ab_gtau.txt 2>&1
cat gpurun_out/ab_gtau.txt
BLURRAST_LIB=$PWD/variants/lib_g1.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_soft.py -x -q 2>&1 | tail -3 > gpurun_out/ab_gtau_parity.log
cat gpurun_out/ab_gtau_parity.log
