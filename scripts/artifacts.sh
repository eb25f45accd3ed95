# Round artifacts on one B200: GPU tests, bench lines (suite 3xTF32 / TF32, reference arm,
# 32/64/128-image shards, GEMM sweep), smoke, the ncu launch list of the plain suite step,
# per-layer ncu metrics of its 20 tile-kernel launches and one `--set full` capture of the stem.
# usage: bash scripts/artifacts.sh TAG        (outputs in gpurun_out/)
TAG=$1
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread,launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,launch__shared_mem_per_block_dynamic"
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>>gpurun_out/bench.err
for b in 32 64 128; do
  timeout 300 python bench.py --batch $b --no-cpu --no-e2e > gpurun_out/bench_b$b.json 2>>gpurun_out/bench.err
done
timeout 300 python bench.py --mode tf32 --no-cpu > gpurun_out/bench_tf32.json 2>>gpurun_out/bench.err
timeout 300 python bench.py --workload gemm --no-cpu --no-e2e > gpurun_out/bench_gemm.json 2>>gpurun_out/bench.err
timeout 200 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1
CMD='python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-graph'
$CMD > gpurun_out/plain.json 2> gpurun_out/plain.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1
ncu --metrics $M --clock-control none -k regex:tile_mma_kernel --launch-skip 60 --launch-count 20 \
  -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tile_mma_kernel --launch-skip 60 \
  --launch-count 1 -o gpurun_out/stem_full_$TAG $CMD > gpurun_out/ncu3.log 2>&1
echo done
