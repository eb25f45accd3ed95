# round-2 i: batched-epilogue ring A/B (boxes of the previous tile may still leave smem while the next are
# written): libpdl_wait0 = round-1 rule, libpdl = ring with 4 buffers, w6 / w8 = 6 / 8 buffers per half
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tiles.py tests/test_gpu_fullsize.py -q > gpurun_out/pytest_r2i.log 2>&1
for lib in libpdl_w6 libpdl_w8; do
PDL_LIB=$PWD/paper_2006_02230_b200/$lib.so timeout 900 python -m pytest tests/test_gpu_parity.py -q >> gpurun_out/pytest_r2i.log 2>&1
done
B='python bench.py --no-cpu --no-e2e --no-extras'
for rep in 1 2; do
for lib in libpdl_wait0 libpdl libpdl_w6 libpdl_w8; do
  PDL_LIB=$PWD/paper_2006_02230_b200/$lib.so timeout 300 $B > gpurun_out/ab_ring_${lib}_$rep.json 2>>gpurun_out/bench_r2i.err
done
done
for lib in libpdl_wait0 libpdl libpdl_w6; do
  PDL_LIB=$PWD/paper_2006_02230_b200/$lib.so timeout 300 $B --batch 32 > gpurun_out/ab_ring_${lib}_b32.json 2>>gpurun_out/bench_r2i.err
done
echo done
