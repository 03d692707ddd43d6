# scratch A/B driver (edited per experiment)
mkdir -p gpurun_out
CONFIGS="C4 C3 C5" bash tools/ab_variants.sh
