# scratch driver (edited per experiment)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in C4 C3; do
timeout 600 python bench.py --config $c --delta 1e-4 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/soft_$c.json
python -c "import json; d=json.load(open('gpurun_out/soft_$c.json')); r=d['roofline']; k=r['kernels_ms']; print('$c soft', round(d['ms_per_step'],3), 'k8 %.2f k9 %.2f k6 %.2f' % (k['k8_soft_fwd'], k['k9_soft_bwd'], k['k6_raster_bwd']), 'terms %.3g items %.3g iters %.3g' % (r['soft_terms_per_launch'], r['soft_items_per_launch'], r['soft_face_iterations_per_launch']), r['kernel'], round(r['frac'],4))"
done
