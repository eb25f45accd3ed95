# round-2 o: layer-5 rule (64-channel k-blocks for BN=64 1x1 convs with >= 128 channels): tests + default bench
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2o.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2o.log
timeout 900 python bench.py > gpurun_out/bench_r2o.json 2> gpurun_out/bench_r2o.err
timeout 300 python bench.py --schedule ranked --no-cpu --no-e2e --no-extras > gpurun_out/bench_ranked_r2o.json 2>> gpurun_out/bench_r2o.err
timeout 300 python bench.py --no-cpu --no-e2e --no-extras > gpurun_out/bench_default2_r2o.json 2>> gpurun_out/bench_r2o.err
echo done
