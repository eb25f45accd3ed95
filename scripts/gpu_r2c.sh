# round-2 c: baseline on the restored tree: GPU tests, default bench line (all sub-objects), shards, smoke
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r2c.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2c.log
timeout 200 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_r2c.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err
timeout 300 python bench.py --batch 32 --no-cpu --no-e2e --no-extras > gpurun_out/bench_b32_r2c.json 2>>gpurun_out/bench_r2c.err
timeout 300 python bench.py --mode tf32 --no-cpu --no-e2e --no-extras > gpurun_out/bench_tf32_r2c.json 2>>gpurun_out/bench_r2c.err
timeout 300 python bench.py --workload gemm --no-cpu --no-e2e > gpurun_out/bench_gemm_r2c.json 2>>gpurun_out/bench_r2c.err
timeout 300 python bench.py --workload pr1 --no-cpu --no-e2e > gpurun_out/bench_pr1_r2c.json 2>>gpurun_out/bench_r2c.err
echo done
