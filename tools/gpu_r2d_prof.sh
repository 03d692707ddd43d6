# round 2, fourth session: final profiles (launch list, ncu --set full of K4/K6) + BASELINE.md section 3 table
mkdir -p gpurun_out
TAG=r2d bash tools/profile_tag.sh
bash tools/baseline_table.sh
