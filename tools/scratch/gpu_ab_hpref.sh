# A/B: BR_K4L_HPREF (next chunk header copied to shared memory by cp.async during the stage), C4 + C3 twice, C5 once,
# then the parity tests on the HPREF library
mkdir -p gpurun_out
for r in 1 2; do
VARIANTS="variants/lib_h0.so variants/lib_h1.so" CONFIGS="C4 C3" bash tools/ab_variants.sh
done > gpurun_out/ab_hpref.txt 2>&1
VARIANTS="variants/lib_h0.so variants/lib_h1.so" CONFIGS="C5" EXTRA="--steps 3 --warmup 3" bash tools/ab_variants.sh >> gpurun_out/ab_hpref.txt 2>&1
cat gpurun_out/ab_hpref.txt
BLURRAST_LIB=$PWD/variants/lib_h1.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_soft.py -x -q 2>&1 | tail -3 > gpurun_out/ab_hpref_parity.log
cat gpurun_out/ab_hpref_parity.log
