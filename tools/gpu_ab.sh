# scratch A/B driver (edited per experiment)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_soft.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
CONFIGS="C4" bash tools/ab_variants.sh
for i in 1 2; do
for v in variants/lib_*.so; do
BLURRAST_LIB=$PWD/$v timeout 600 python bench.py --config C4 --delta 1e-4 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=r['kernels_ms']; print('$v C4 soft', round(d['ms_per_step'],3), 'k4 %.2f k8 %.2f k9 %.2f' % (k['k4_raster_fwd'], k['k8_soft_fwd'], k['k9_soft_bwd']))"
done
done
