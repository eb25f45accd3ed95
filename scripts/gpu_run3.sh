timeout 300 python scripts/probe_split_debug.py > gpurun_out/split_debug.log 2>&1
PDL_NO_PDL=1 timeout 300 python scripts/probe_split_debug.py > gpurun_out/split_debug_nopdl.log 2>&1
timeout 900 python -m pytest tests/test_gpu_gemm_epilogue.py -q > gpurun_out/pytest_epi.log 2>&1
for fam in gemm halo stem resident splitk gemm_splitk host simt layout; do
  for tool in memcheck synccheck racecheck; do
    echo "== $fam $tool" >> gpurun_out/sanitizer.log
    t0=$(date +%s)
    timeout 300 compute-sanitizer --tool $tool --error-exitcode 99 python scripts/sanitize_case.py $fam > gpurun_out/san_tmp.log 2>&1
    rc=$?
    tail -4 gpurun_out/san_tmp.log >> gpurun_out/sanitizer.log
    echo "rc=$rc secs=$(( $(date +%s) - t0 ))" >> gpurun_out/sanitizer.log
  done
done
