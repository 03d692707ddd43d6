# session-3 first call: GPU tests, smoke, default bench line, r2b profile (launch list + ncu full of K4/K6)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu_s3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_s3.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s3.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_s3.log
timeout 600 python bench.py > gpurun_out/bench_s3.json 2> gpurun_out/bench_s3.err
bash tools/profile_r2b.sh > gpurun_out/profile_r2b.log 2>&1
