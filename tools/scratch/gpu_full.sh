# full GPU test suite + the default bench line (both arms) on one box
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu_full.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for v in variants/lib_r1.so variants/lib_cur.so; do BLURRAST_LIB=$PWD/$v python tools/time_raster.py C4 >> gpurun_out/tr_ab.log 2>&1; done
