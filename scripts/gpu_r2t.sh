# round-2 t: TF32 rules + cached box search: tests and A/B against the previous library
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2t.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2t.log
B='python bench.py --no-cpu --no-e2e --no-extras'
for lib in libpdl_prev libpdl; do
  for b in 256 32 28; do
    PDL_LIB=$PWD/paper_2006_02230_b200/$lib.so timeout 300 $B --mode tf32 --batch $b > gpurun_out/ab_t_${lib}_tf32_b$b.json 2>>gpurun_out/bench_r2t.err
  done
  for b in 256 32; do
    PDL_LIB=$PWD/paper_2006_02230_b200/$lib.so timeout 300 $B --batch $b > gpurun_out/ab_t_${lib}_b$b.json 2>>gpurun_out/bench_r2t.err
  done
done
echo done
