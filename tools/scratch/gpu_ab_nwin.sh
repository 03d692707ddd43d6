# A/B: BR_K4L_NWIN (bin sizes of 32 chunks per load), C4 + C3 twice, then the parity tests
mkdir -p gpurun_out
for r in 1 2; do
VARIANTS="variants/lib_nw0.so variants/lib_nw1.so" CONFIGS="C4 C3" bash tools/ab_variants.sh
done > gpurun_out/ab_nwin.txt 2>&1
cat gpurun_out/ab_nwin.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3 > gpurun_out/ab_nwin_parity.log
cat gpurun_out/ab_nwin_parity.log
