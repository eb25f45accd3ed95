for lib in libpdl_prev libpdl; do
  echo "== $lib"
  PDL_LIB=$PWD/paper_2006_02230_b200/$lib.so timeout 300 python scripts/time_layer.py 32 tf32 8 9 14 17 20 16
done > gpurun_out/tf32_b32_iso.log 2>&1
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_sanitizer.py tests/test_gpu_parity.py -q > gpurun_out/pytest_r2s.log 2>&1
echo done
