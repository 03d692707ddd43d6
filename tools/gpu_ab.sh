# scratch A/B driver (edited per experiment)
mkdir -p gpurun_out
for i in 1 2 3; do CONFIGS="C4" bash tools/ab_variants.sh; done
