# round-2 m: constant-bank warm-up + split-K exchange (coalesced partial layout, two-range register path)
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2m.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2m.log
B='python bench.py --no-cpu --no-e2e --no-extras'
for rep in 1 2; do
for lib in libpdl_head libpdl; do
  PDL_LIB=$PWD/paper_2006_02230_b200/$lib.so timeout 300 $B --batch 32 > gpurun_out/ab_m_${lib}_b32_$rep.json 2>>gpurun_out/bench_r2m.err
  PDL_LIB=$PWD/paper_2006_02230_b200/$lib.so timeout 300 $B --batch 28 > gpurun_out/ab_m_${lib}_b28_$rep.json 2>>gpurun_out/bench_r2m.err
done
done
for lib in libpdl_head libpdl; do
  PDL_LIB=$PWD/paper_2006_02230_b200/$lib.so timeout 300 $B > gpurun_out/ab_m_${lib}_b256.json 2>>gpurun_out/bench_r2m.err
  PDL_LIB=$PWD/paper_2006_02230_b200/$lib.so timeout 300 python bench.py --workload gemm --no-cpu --no-e2e > gpurun_out/ab_m_${lib}_gemm.json 2>>gpurun_out/bench_r2m.err
  PDL_LIB=$PWD/paper_2006_02230_b200/$lib.so timeout 300 python bench.py --workload pr1 --no-cpu --no-e2e > gpurun_out/ab_m_${lib}_pr1.json 2>>gpurun_out/bench_r2m.err
done
PDL_LIB=$PWD/paper_2006_02230_b200/libpdl_trace.so timeout 600 python scripts/probe_timeline.py 32 16 20 6 17 pr1 g64,64,64 g3136,64,576 > gpurun_out/timeline_r2m.log 2>&1
echo done
