timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu6.log 2>&1
bash scripts/ab_suite_libs.sh "scripts/libpdl_r1q.so paper_2006_02230_b200/libpdl.so" 2 > gpurun_out/ab_fence.log 2>&1
timeout 300 python bench.py --no-extras --no-cpu --no-e2e --m-fastest > gpurun_out/bench_mfast.json 2>&1
timeout 300 python bench.py --no-extras --no-cpu --no-e2e --batch 32 > gpurun_out/bench_b32.json 2>&1
timeout 300 python bench.py --no-extras --no-cpu --no-e2e --batch 32 --m-fastest > gpurun_out/bench_b32_mfast.json 2>&1
