# round 2, fifth session, final code (WCLR on): suite + smoke + bench + profiles (tools/gpu_r2e.sh), then the checked build
bash tools/gpu_r2e.sh
bash tools/checked_build.sh
