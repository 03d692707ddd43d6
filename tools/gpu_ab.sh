# scratch A/B driver (edited per experiment)
mkdir -p gpurun_out
for i in 1 2; do CONFIGS="C4 C3" bash tools/ab_variants.sh; done
