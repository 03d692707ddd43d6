# round-2 measurement call: GPU tests, smoke, BASELINE.md section 3 bench lines (C1-C5), soft C4 line
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
bash tools/baseline_table.sh > gpurun_out/baseline_table.log 2>&1
timeout 900 python bench.py --delta 1e-4 --no-cpu-baseline > gpurun_out/bench_c4_soft.json 2> gpurun_out/bench_c4_soft.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
