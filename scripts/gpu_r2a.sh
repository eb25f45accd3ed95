# round-2 baseline on the restored tree: GPU tests, default bench line, 32-image shard, TF32 suite
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r2a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2a.log
timeout 900 python bench.py > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err
timeout 300 python bench.py --batch 32 --no-cpu --no-e2e --no-extras > gpurun_out/bench_b32_r2a.json 2>>gpurun_out/bench_r2a.err
timeout 300 python bench.py --mode tf32 --no-cpu --no-e2e --no-extras > gpurun_out/bench_tf32_r2a.json 2>>gpurun_out/bench_r2a.err
timeout 200 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_r2a.log 2>&1
