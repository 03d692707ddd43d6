# round 2, fifth session: last check of the committed tree (all variant flags at their defaults): GPU suite, smoke, default bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/r2e_last_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2e_last_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r2e_last_bench_C4.json 2> gpurun_out/r2e_last_bench_C4.err
cat gpurun_out/r2e_last_pytest_gpu.log; tail -2 gpurun_out/r2e_last_smoke.log; head -c 330 gpurun_out/r2e_last_bench_C4.json
