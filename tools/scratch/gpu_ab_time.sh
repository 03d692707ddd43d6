# kernel-time A/B of library variants on a config (tools/time_raster.py)
mkdir -p gpurun_out
for v in ${VARIANTS:-variants/lib_*.so}; do echo "== $v" >> gpurun_out/tr_ab.log; BLURRAST_LIB=$PWD/$v timeout 300 python tools/time_raster.py ${CFG:-C4} >> gpurun_out/tr_ab.log 2>&1; done
