# Checked build (-DBR_CHECKED: shared-memory index invariants of the raster kernels tested at run time, a violation
# raises BLUR_ST_EINTERNAL) run over the GPU test suite (the parity tests assert that no call raised BLUR_ST_EINTERNAL; BLURRAST_CHECK=1 would also turn the expected
# bin overflows of the auto-sizing first forward into errors), for
# the default forward and the super-grouped A/B -- the memory-safety evidence in place of compute-sanitizer, which
# this pool has closed.  Needs variants/lib_checked.so (python tools/build_variants.py checked:BR_CHECKED).
mkdir -p gpurun_out
{
  echo "== checked build, default kernels"; BLURRAST_LIB=$PWD/variants/lib_checked.so timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
  echo "== checked build, BLURRAST_FWD=sg"; BLURRAST_FWD=sg BLURRAST_LIB=$PWD/variants/lib_checked.so timeout 900 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -3
  echo "== checked build, sanitize_small"; BLURRAST_LIB=$PWD/variants/lib_checked.so timeout 600 python tools/sanitize_small.py 2>&1 | tail -5
} > gpurun_out/checked_build.log 2>&1
cat gpurun_out/checked_build.log
