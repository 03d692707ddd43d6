# one bench line per config at 1 GPU (C1-C3 as CUDA graphs: launch-bound), each
# with its CPU-oracle baseline; writes gpurun_out/table_<cfg>.json and prints the markdown rows.
mkdir -p gpurun_out
for c in C1 C2 C3; do
  timeout 900 python bench.py --config $c --graph --steps 50 --warmup 5 --cpu-seconds 10 > gpurun_out/table_$c.json 2> gpurun_out/table_$c.err
done
timeout 900 python bench.py --config C4 --steps 20 --warmup 5 --cpu-seconds 12 > gpurun_out/table_C4.json 2> gpurun_out/table_C4.err
timeout 1500 python bench.py --config C5 --steps 3 --warmup 3 --cpu-seconds 30 > gpurun_out/table_C5.json 2> gpurun_out/table_C5.err
python tools/table_rows.py gpurun_out/table_C1.json gpurun_out/table_C2.json gpurun_out/table_C3.json \
    gpurun_out/table_C4.json gpurun_out/table_C5.json > gpurun_out/table_rows.md
cat gpurun_out/table_rows.md
for c in C2 C3; do
  timeout 900 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/table_${c}_eager.json 2> gpurun_out/table_${c}_eager.err
done
timeout 900 python bench.py --delta 1e-4 --no-cpu-baseline > gpurun_out/table_C4_soft.json 2> gpurun_out/table_C4_soft.err
python tools/table_rows.py gpurun_out/table_C2_eager.json gpurun_out/table_C3_eager.json gpurun_out/table_C4_soft.json > gpurun_out/table_rows_extra.md
cat gpurun_out/table_rows_extra.md
