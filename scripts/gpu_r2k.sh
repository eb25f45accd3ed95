timeout 600 python -m pytest tests/test_gpu_stem_compact.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_sanitizer.py -q > gpurun_out/pytest_r2k.log 2>&1
for lib in libpdl_head libpdl; do
  echo "== $lib"
  PDL_LIB=$PWD/paper_2006_02230_b200/$lib.so timeout 300 python scripts/time_layer.py 256 3xtf32 1 1 3
  PDL_LIB=$PWD/paper_2006_02230_b200/$lib.so timeout 300 python scripts/time_layer.py 256 tf32 1
  PDL_LIB=$PWD/paper_2006_02230_b200/$lib.so timeout 300 python scripts/time_layer.py 32 3xtf32 1
done > gpurun_out/stem_iso.log 2>&1
echo done
