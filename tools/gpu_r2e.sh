# round 2, fifth session: GPU suite + smoke + default bench + profiles (launch list, ncu --set full K4/K6)
# on the final code (after BR_K4L_EKEEP / BR_K4L_R48), then the C3 and C5 bench lines
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/r2e_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2e_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r2e_bench_C4.json 2> gpurun_out/r2e_bench_C4.err
TAG=r2e bash tools/profile_tag.sh
timeout 900 python bench.py --config C3 --graph --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2e_bench_C3.json 2> gpurun_out/r2e_bench_C3.err
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2e_bench_C5.json 2> gpurun_out/r2e_bench_C5.err
cat gpurun_out/r2e_pytest_gpu.log; tail -1 gpurun_out/r2e_smoke.log
for f in C4 C3 C5; do head -c 330 gpurun_out/r2e_bench_$f.json; echo; done
