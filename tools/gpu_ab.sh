# scratch driver
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200; done
