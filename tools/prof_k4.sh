# ncu --set full of K4/K6 on C4 (one warm-up step), plus per-line instruction tables.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CMD1="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD1 > gpurun_out/plain1.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k4_raster_fwd|k6_raster_bwd" -s 4 -c 2 \
    -o gpurun_out/prof_k4 $CMD1 > gpurun_out/ncu_full.log 2>&1
python tools/ncu_lines2.py gpurun_out/prof_k4.ncu-rep k4_raster_fwd 60 > gpurun_out/lines_k4.txt 2>&1
python tools/ncu_lines2.py gpurun_out/prof_k4.ncu-rep k6_raster_bwd 60 > gpurun_out/lines_k6.txt 2>&1
echo done
