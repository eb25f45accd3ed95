# round-2 b: new tests (families / canaries, compact stem), bench with compact-stem sub-objects
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r2b.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2b.log
timeout 900 python bench.py > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err
