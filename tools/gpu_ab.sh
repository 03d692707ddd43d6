# scratch A/B driver (edited per experiment)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_soft.py -m gpu -x -q 2>&1 | tail -3
for c in C4 C3 C2; do
timeout 600 python bench.py --config $c --delta 1e-4 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c soft', round(d['ms_per_step'],3), r['kernels_ms'])"
done
