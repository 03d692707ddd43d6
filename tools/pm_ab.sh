# order (i) (k4i_raster_fwd, BLURRAST_FWD=pixmajor) variants: kernel times on C4/C3 + one ncu --set full capture
mkdir -p gpurun_out
for v in ${VARIANTS:-pmkp4 pmkp2 pmkp4nb128}; do echo "== $v"; BLURRAST_FWD=pixmajor BLURRAST_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/time_raster.py C4 2>&1 | head -1; BLURRAST_FWD=pixmajor BLURRAST_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/time_raster.py C3 2>&1 | head -1; done
BLURRAST_FWD=pixmajor BLURRAST_LIB=$PWD/variants/lib_${NCU_V:-pmkp4}.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:k4i_raster_fwd -s 1 -c 1 -o gpurun_out/prof_pm_c4 python tools/time_raster.py C4 1 > gpurun_out/ncu_pm.log 2>&1; echo ncu=$?
