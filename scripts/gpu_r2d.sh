# round-2 d: ncu evidence on the restored tree: launch list of the plain suite step (256 and 32 images),
# per-layer metrics, GEMM sweep launch list + metrics, one --set full capture of the dominant kernel
TAG=r2d
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread,launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,launch__shared_mem_per_block_dynamic"
CMD='python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-graph --no-extras'
$CMD > gpurun_out/plain_$TAG.json 2> gpurun_out/plain_$TAG.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu1.log 2>&1
ncu --metrics $M --clock-control none -k regex:tile_mma_kernel --launch-skip 60 --launch-count 20 \
  -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu2.log 2>&1
CMD32="$CMD --batch 32"
$CMD32 > gpurun_out/plain_b32_$TAG.json 2>> gpurun_out/plain_$TAG.err && \
ncu --metrics $M --clock-control none -k regex:tile_mma_kernel --launch-skip 60 --launch-count 20 \
  -o gpurun_out/prof_b32_$TAG $CMD32 > gpurun_out/ncu3.log 2>&1
CMDG='python bench.py --workload gemm --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph'
$CMDG > gpurun_out/plain_gemm_$TAG.json 2>> gpurun_out/plain_$TAG.err && \
ncu --metrics $M --clock-control none -k regex:tile_mma_kernel -c 400 \
  -o gpurun_out/prof_gemm_$TAG $CMDG > gpurun_out/ncu4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tile_mma_kernel --launch-skip 62 \
  --launch-count 1 -o gpurun_out/l03_full_$TAG $CMD > gpurun_out/ncu5.log 2>&1
echo done
