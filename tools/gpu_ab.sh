# scratch A/B driver (edited per experiment)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_soft.py -m gpu -x -q 2>&1 | tail -2
for v in variants/lib_*.so; do
for c in C4 C3; do
BLURRAST_LIB=$PWD/$v timeout 600 python bench.py --config $c --delta 1e-4 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=r['kernels_ms']; print('$v $c soft', round(d['ms_per_step'],3), 'k8 %.2f k9 %.2f' % (k['k8_soft_fwd'], k['k9_soft_bwd']))"
done
BLURRAST_LIB=$PWD/$v timeout 900 python bench.py --config C5 --delta 1e-4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=r['kernels_ms']; print('$v C5 soft', round(d['ms_per_step'],3), 'k8 %.2f k9 %.2f' % (k['k8_soft_fwd'], k['k9_soft_bwd']))"
done
