# round 2, fourth session: GPU suite + smoke + default bench on a fresh box
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -25 > gpurun_out/r2d_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2d_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r2d_bench_C4.log 2>&1
tail -3 gpurun_out/r2d_pytest_gpu.log; tail -1 gpurun_out/r2d_smoke.log; tail -1 gpurun_out/r2d_bench_C4.log
