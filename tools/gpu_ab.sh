# scratch driver (edited per experiment)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python studies/recovery.py > gpurun_out/recovery.log 2> gpurun_out/recovery.err; echo recovery=$?
cp studies/recovery_r1.md gpurun_out/recovery_r1.md 2>/dev/null; tail -12 gpurun_out/recovery.log
