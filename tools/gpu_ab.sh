# scratch driver: re-run the studies with the current kernels
mkdir -p gpurun_out
for s in ablation segmentation soft_approx; do
  timeout 1200 python studies/$s.py > gpurun_out/study_$s.md 2> gpurun_out/study_$s.err; echo $s=$?
done
