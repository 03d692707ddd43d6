# end-of-session GPU call: GPU suite + smoke (default build), the A/B forwards over the parity tests, the checked
# build, ncu profile of K4/K6 and the bench lines of every config
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_final.log
for fw in pixmajor sg; do echo "== BLURRAST_FWD=$fw" >> gpurun_out/variants_parity.log; BLURRAST_FWD=$fw timeout 900 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -2 >> gpurun_out/variants_parity.log; done
bash tools/checked_build.sh > /dev/null 2>&1
bash tools/profile_r2b.sh > gpurun_out/profile_r2b.log 2>&1
bash tools/baseline_table.sh > gpurun_out/baseline_table.log 2>&1
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py --config C5 --delta 1e-4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/table_C5_soft.json 2> gpurun_out/table_C5_soft.err
