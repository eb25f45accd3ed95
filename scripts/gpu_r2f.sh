# round-2 f: GPU tests with the new tile tests, tile-shape probe, L2 fetch granularity probe, traces at 32 images
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2f.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2f.log
timeout 900 python scripts/probe_tile_shapes.py 256 3xtf32 > gpurun_out/tile_shapes_256.log 2>&1
timeout 900 python scripts/probe_tile_shapes.py 32 3xtf32 > gpurun_out/tile_shapes_32.log 2>&1
timeout 900 python scripts/probe_tile_shapes.py 256 tf32 > gpurun_out/tile_shapes_256_tf32.log 2>&1
timeout 600 python scripts/probe_l2_fetch.py > gpurun_out/l2_fetch.log 2>&1
N=32 PDL_LIB=$PWD/paper_2006_02230_b200/libpdl_trace.so timeout 600 python scripts/probe_trace.py 16 6 20 2 13 > gpurun_out/trace_b32.log 2>&1
PDL_LIB=$PWD/paper_2006_02230_b200/libpdl_trace.so timeout 600 python scripts/probe_trace.py 3 8 4 1 > gpurun_out/trace_b256.log 2>&1
echo done
