timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu2.log 2>&1
timeout 900 python scripts/probe_split_bug.py > gpurun_out/split_bug.log 2>&1
for fam in gemm halo stem resident splitk gemm_splitk host simt layout; do
  for tool in memcheck synccheck racecheck; do
    echo "== $fam $tool" >> gpurun_out/sanitizer.log
    /usr/bin/time -f "%e s" timeout 300 compute-sanitizer --tool $tool --error-exitcode 99 python scripts/sanitize_case.py $fam >> gpurun_out/sanitizer.log 2>&1
    echo "rc=$?" >> gpurun_out/sanitizer.log
  done
done
