# scratch driver (edited per experiment)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py 2>&1 | tail -1 | cut -c1-300
