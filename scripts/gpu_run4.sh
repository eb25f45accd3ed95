for v in 1 2; do
  echo "=== halo$v" >> gpurun_out/halofix.log
  PDL_LIB=$PWD/scripts/libpdl_halo$v.so timeout 300 python scripts/probe_split_debug.py >> gpurun_out/halofix.log 2>&1
  PDL_LIB=$PWD/scripts/libpdl_halo$v.so timeout 600 python scripts/probe_split_bug.py >> gpurun_out/halofix.log 2>&1
done
