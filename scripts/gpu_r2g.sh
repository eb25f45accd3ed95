# round-2 g: wave-aware box search + non-halo full tiles + single-wave split-K: tests and A/B
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2g.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2g.log
B='python bench.py --no-cpu --no-e2e --no-extras'
timeout 300 $B > gpurun_out/ab_g_new_1.json 2>>gpurun_out/bench_r2g.err
timeout 300 $B --single-image-tiles > gpurun_out/ab_g_old_1.json 2>>gpurun_out/bench_r2g.err
timeout 300 $B --batch 32 > gpurun_out/ab_g_new_b32.json 2>>gpurun_out/bench_r2g.err
timeout 300 $B --batch 32 --single-image-tiles > gpurun_out/ab_g_old_b32.json 2>>gpurun_out/bench_r2g.err
timeout 300 $B --batch 64 > gpurun_out/ab_g_new_b64.json 2>>gpurun_out/bench_r2g.err
timeout 300 $B --batch 128 > gpurun_out/ab_g_new_b128.json 2>>gpurun_out/bench_r2g.err
timeout 300 $B --mode tf32 > gpurun_out/ab_g_new_tf32.json 2>>gpurun_out/bench_r2g.err
timeout 300 $B --mode tf32 --single-image-tiles > gpurun_out/ab_g_old_tf32.json 2>>gpurun_out/bench_r2g.err
timeout 900 python bench.py > gpurun_out/bench_r2g.json 2>>gpurun_out/bench_r2g.err
echo done
