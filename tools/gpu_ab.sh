# scratch A/B driver (edited per experiment)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do CONFIGS="C4 C3" bash tools/ab_variants.sh; done
