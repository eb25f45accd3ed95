timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu5.log 2>&1
bash scripts/ab_suite_libs.sh "scripts/libpdl_r1q.so paper_2006_02230_b200/libpdl.so" 2 > gpurun_out/ab_fence.log 2>&1
