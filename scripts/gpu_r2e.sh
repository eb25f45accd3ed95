# round-2 e: multi-image box tile search -- GPU tests, then same-box A/B against the round-1 geometry
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2e.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2e.log
B='python bench.py --no-cpu --no-e2e --no-extras'
for rep in 1 2; do
  timeout 300 $B > gpurun_out/ab_tiles_new_$rep.json 2>>gpurun_out/bench_r2e.err
  timeout 300 $B --single-image-tiles > gpurun_out/ab_tiles_old_$rep.json 2>>gpurun_out/bench_r2e.err
done
timeout 300 $B --batch 32 > gpurun_out/ab_tiles_new_b32.json 2>>gpurun_out/bench_r2e.err
timeout 300 $B --batch 32 --single-image-tiles > gpurun_out/ab_tiles_old_b32.json 2>>gpurun_out/bench_r2e.err
timeout 300 $B --mode tf32 > gpurun_out/ab_tiles_new_tf32.json 2>>gpurun_out/bench_r2e.err
timeout 300 $B --mode tf32 --single-image-tiles > gpurun_out/ab_tiles_old_tf32.json 2>>gpurun_out/bench_r2e.err
echo done
