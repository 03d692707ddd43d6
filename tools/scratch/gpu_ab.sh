# scratch A/B driver (edited per experiment)
mkdir -p gpurun_out
CONFIGS="C4 C3" bash tools/ab_variants.sh
for v in variants/lib_def.so variants/lib_k9m4.so; do
BLURRAST_LIB=$PWD/$v timeout 600 python bench.py --config C4 --delta 1e-4 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=r['kernels_ms']; print('$v C4 soft', round(d['ms_per_step'],3), 'k8 %.2f k9 %.2f' % (k['k8_soft_fwd'], k['k9_soft_bwd']))"
done
