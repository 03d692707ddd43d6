# A/B: occupancy / group size / split sweep of the lean K4 after WCLR (C4 twice, C3 and C5 once)
mkdir -p gpurun_out
{
for r in 1 2; do
VARIANTS="variants/lib_h0.so variants/lib_m4.so variants/lib_m4s.so variants/lib_hs3.so variants/lib_hs4.so" CONFIGS="C4" bash tools/ab_variants.sh
done
VARIANTS="variants/lib_h0.so variants/lib_m4.so variants/lib_m4s.so variants/lib_hs3.so variants/lib_hs4.so" CONFIGS="C3" bash tools/ab_variants.sh
VARIANTS="variants/lib_h0.so variants/lib_m4s.so variants/lib_hs3.so" CONFIGS="C5" EXTRA="--steps 3 --warmup 3" bash tools/ab_variants.sh
} > gpurun_out/ab_sweep.txt 2>&1
cat gpurun_out/ab_sweep.txt
