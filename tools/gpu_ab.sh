# scratch A/B driver (edited per experiment)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_soft.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --delta 1e-4 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('soft C4', round(d['ms_per_step'],2), r['kernels_ms'])"
timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('hard C4', round(d['ms_per_step'],3), r['kernels_ms'] if 'kernels_ms' in r else (r['fwd_raster_ms'], r['bwd_raster_ms']))"
