mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/pt_dist.log 2>&1; tail -3 gpurun_out/pt_dist.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err
timeout 1500 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err
