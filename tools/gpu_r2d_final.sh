# round 2, fourth session: final GPU suite + smoke on the committed code, reference arm, C5 soft line, default bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/r2d_final_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2d_final_smoke.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py --config C5 --delta 1e-4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/table_C5_soft.json 2> gpurun_out/table_C5_soft.err
timeout 600 python bench.py > gpurun_out/r2d_final_bench_C4.json 2> gpurun_out/r2d_final_bench_C4.err
cat gpurun_out/r2d_final_pytest_gpu.log; tail -1 gpurun_out/r2d_final_smoke.log; tail -c 400 gpurun_out/bench_ref.json; tail -c 300 gpurun_out/table_C5_soft.json; tail -c 300 gpurun_out/r2d_final_bench_C4.json
