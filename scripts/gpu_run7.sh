for b in 256 32 28; do
  timeout 1500 python scripts/sweep_variants.py --batch $b --out gpurun_out/sweep_r2_b$b.json > gpurun_out/sweep_b$b.log 2>&1
done
