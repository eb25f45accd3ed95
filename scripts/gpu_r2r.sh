# round-2 r: TF32 rules (64-channel k-blocks for spatial BN=256 layers; BN=128 when 256-column tiles leave SMs idle)
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2r.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2r.log
B='python bench.py --no-cpu --no-e2e --no-extras --mode tf32'
for lib in libpdl_prev libpdl; do
  for b in 256 32 28; do
    PDL_LIB=$PWD/paper_2006_02230_b200/$lib.so timeout 300 $B --batch $b > gpurun_out/ab_r_${lib}_tf32_b$b.json 2>>gpurun_out/bench_r2r.err
  done
done
echo done
