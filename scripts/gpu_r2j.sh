# round-2 j: stem with 8 staging warps (two sets alternate k-blocks) and 4 epilogue warps: tests, A/B vs HEAD
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2j.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2j.log
B='python bench.py --no-cpu --no-e2e --no-extras'
for rep in 1 2; do
for lib in libpdl_head libpdl; do
  PDL_LIB=$PWD/paper_2006_02230_b200/$lib.so timeout 300 $B > gpurun_out/ab_stem_${lib}_$rep.json 2>>gpurun_out/bench_r2j.err
done
done
for lib in libpdl_head libpdl; do
  PDL_LIB=$PWD/paper_2006_02230_b200/$lib.so timeout 300 $B --batch 32 > gpurun_out/ab_stem_${lib}_b32.json 2>>gpurun_out/bench_r2j.err
  PDL_LIB=$PWD/paper_2006_02230_b200/$lib.so timeout 300 $B --mode tf32 > gpurun_out/ab_stem_${lib}_tf32.json 2>>gpurun_out/bench_r2j.err
done
echo done
