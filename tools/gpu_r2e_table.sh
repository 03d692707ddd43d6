# round 2, fifth session: the remaining BASELINE.md section 3 lines on the final code (C1/C2 graphs, eager C2/C3, soft C4/C5)
mkdir -p gpurun_out
for c in C1 C2; do
  timeout 900 python bench.py --config $c --graph --steps 50 --warmup 5 --cpu-seconds 10 > gpurun_out/table_$c.json 2> gpurun_out/table_$c.err
done
for c in C2 C3; do
  timeout 900 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/table_${c}_eager.json 2> gpurun_out/table_${c}_eager.err
done
timeout 900 python bench.py --delta 1e-4 --no-cpu-baseline > gpurun_out/table_C4_soft.json 2> gpurun_out/table_C4_soft.err
timeout 900 python bench.py --config C5 --delta 1e-4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/table_C5_soft.json 2> gpurun_out/table_C5_soft.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python tools/table_rows.py gpurun_out/table_C1.json gpurun_out/table_C2.json gpurun_out/table_C2_eager.json gpurun_out/table_C3_eager.json gpurun_out/table_C4_soft.json gpurun_out/table_C5_soft.json
tail -c 300 gpurun_out/bench_ref.json
