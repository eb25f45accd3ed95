# round-2 d: ncu evidence: launch list of the plain suite step (256 images), per-layer metrics at 256 and
# 32 images, GEMM sweep metrics, one --set full capture of the dominant kernel (L03).  Reports are exported
# to CSV on the box (gpurun_out/ is capped at 64 MiB).
TAG=${1:-r2d}
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread,launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,launch__shared_mem_per_block_dynamic"
T=/tmp/ncu_$TAG; mkdir -p $T
CMD='python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-graph --no-extras'
$CMD > gpurun_out/plain_$TAG.json 2> gpurun_out/plain_$TAG.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu1.log 2>&1
ncu --metrics $M --clock-control none -k regex:tile_mma_kernel --launch-skip 60 --launch-count 20 \
  -o $T/prof $CMD > gpurun_out/ncu2.log 2>&1
ncu -i $T/prof.ncu-rep --page raw --csv > gpurun_out/prof_$TAG.csv
CMD32="$CMD --batch 32"
ncu --metrics $M --clock-control none -k regex:tile_mma_kernel --launch-skip 60 --launch-count 20 \
  -o $T/prof_b32 $CMD32 > gpurun_out/ncu3.log 2>&1
ncu -i $T/prof_b32.ncu-rep --page raw --csv > gpurun_out/prof_b32_$TAG.csv
CMDG='python bench.py --workload gemm --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph'
$CMDG > gpurun_out/plain_gemm_$TAG.json 2>> gpurun_out/plain_$TAG.err && \
ncu --metrics $M --clock-control none -k regex:tile_mma_kernel -c 600 \
  -o $T/prof_gemm $CMDG > gpurun_out/ncu4.log 2>&1
ncu -i $T/prof_gemm.ncu-rep --page raw --csv > gpurun_out/prof_gemm_$TAG.csv
ncu --set full --clock-control none --import-source on -k regex:tile_mma_kernel --launch-skip 62 \
  --launch-count 1 -o $T/l03_full $CMD > gpurun_out/ncu5.log 2>&1
ncu -i $T/l03_full.ncu-rep --page raw --csv > gpurun_out/l03_full_$TAG.csv
ncu -i $T/l03_full.ncu-rep --page details --csv > gpurun_out/l03_full_details_$TAG.csv
ls -la $T > gpurun_out/ncu_sizes_$TAG.log
echo done
