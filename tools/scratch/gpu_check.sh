set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench_c4.log 2>&1; echo bench=$?
timeout 600 python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo bench3=$?
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench_c4.log; tail -1 gpurun_out/bench_c3.log
