# Round artifacts on one B200 (outputs in gpurun_out/, summarised into profiles/ by scripts/summarize_ncu.py):
# GPU tests, smoke, bench lines (default with every sub-object; reference arm; 32/64/128-image shards; TF32
# suite; GEMM sweep; PR1), the ncu launch list of the plain suite step, per-layer ncu metrics at 256 and 32
# images, one profiled launch per GEMM shape + PR1, and one `--set full` capture of the dominant kernel.
# ncu reports are exported to CSV on the box (gpurun_out/ is capped at 64 MiB).
# usage: bash scripts/artifacts.sh TAG
TAG=$1
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread,launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,launch__shared_mem_per_block_dynamic"
T=/tmp/ncu_$TAG; mkdir -p $T
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 200 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_$TAG.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>>gpurun_out/bench_$TAG.err
for b in 32 64 128; do
  timeout 300 python bench.py --batch $b --no-cpu --no-e2e --no-extras > gpurun_out/bench_b${b}_$TAG.json 2>>gpurun_out/bench_$TAG.err
done
timeout 300 python bench.py --mode tf32 --no-cpu --no-extras > gpurun_out/bench_tf32_$TAG.json 2>>gpurun_out/bench_$TAG.err
timeout 300 python bench.py --workload gemm --no-cpu --no-e2e > gpurun_out/bench_gemm_$TAG.json 2>>gpurun_out/bench_$TAG.err
timeout 300 python bench.py --workload pr1 --no-cpu --no-e2e > gpurun_out/bench_pr1_$TAG.json 2>>gpurun_out/bench_$TAG.err
CMD='python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-graph --no-extras'
$CMD > gpurun_out/plain_$TAG.json 2> gpurun_out/plain_$TAG.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu1.log 2>&1
ncu --metrics $M --clock-control none -k regex:tile_mma_kernel --launch-skip 60 --launch-count 20 \
  -o $T/prof $CMD > gpurun_out/ncu2.log 2>&1
ncu -i $T/prof.ncu-rep --page raw --csv > gpurun_out/prof_$TAG.csv
ncu --metrics $M --clock-control none -k regex:tile_mma_kernel --launch-skip 60 --launch-count 20 \
  -o $T/prof_b32 $CMD --batch 32 > gpurun_out/ncu3.log 2>&1
ncu -i $T/prof_b32.ncu-rep --page raw --csv > gpurun_out/prof_b32_$TAG.csv
for mode in 3xtf32 tf32; do
  python scripts/ncu_gemm_case.py $mode > gpurun_out/gemm_case_$mode.log 2>&1 && \
  ncu --profile-from-start off --metrics $M --clock-control none -k regex:tile_mma_kernel \
    -o $T/prof_gemm_$mode python scripts/ncu_gemm_case.py $mode > gpurun_out/ncu4_$mode.log 2>&1
  ncu -i $T/prof_gemm_$mode.ncu-rep --page raw --csv > gpurun_out/prof_gemm_${mode}_$TAG.csv
done
# the dominant kernel of the step (launch 60 = the stem, 62 = layer 3 of the profiled step)
ncu --set full --clock-control none --import-source on -k regex:tile_mma_kernel --launch-skip 60 \
  --launch-count 1 -o $T/dom_full $CMD > gpurun_out/ncu5.log 2>&1
ncu -i $T/dom_full.ncu-rep --page raw --csv > gpurun_out/dom_full_$TAG.csv
ncu -i $T/dom_full.ncu-rep --page details --csv > gpurun_out/dom_full_details_$TAG.csv
ls -la $T > gpurun_out/ncu_sizes_$TAG.log
echo done
