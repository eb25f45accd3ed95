# round-2 h: L2 prefetch distance A/B (PDL_PF = units ahead per CTA)
B='python bench.py --no-cpu --no-e2e --no-extras'
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tiles.py tests/test_gpu_splitk.py -q > gpurun_out/pytest_pf4.log 2>&1
PDL_PF=4 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tiles.py tests/test_gpu_splitk.py -q >> gpurun_out/pytest_pf4.log 2>&1
for pf in 0 2 4 8 0 4; do
  PDL_PF=$pf timeout 300 $B > gpurun_out/ab_pf${pf}_$RANDOM.json 2>>gpurun_out/bench_r2h.err
done
for pf in 0 4 8; do
  PDL_PF=$pf timeout 300 $B --batch 32 > gpurun_out/ab_b32_pf${pf}.json 2>>gpurun_out/bench_r2h.err
  PDL_PF=$pf timeout 300 $B --mode tf32 > gpurun_out/ab_tf32_pf${pf}.json 2>>gpurun_out/bench_r2h.err
done
echo done
