# scratch A/B driver (edited per experiment)
mkdir -p gpurun_out
for v in variants/lib_*.so; do
for c in C4 C3; do
BLURRAST_LIB=$PWD/$v timeout 600 python bench.py --config $c --delta 1e-4 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=r['kernels_ms']; print('$v $c soft', round(d['ms_per_step'],3), 'k8 %.2f k9 %.2f' % (k['k8_soft_fwd'], k['k9_soft_bwd']))"
done
done
