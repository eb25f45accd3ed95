# round-2 n: variant sweep on the round-2 kernels (tile box, halo, split, order dimensions), 256 and 32 images
timeout 2400 python scripts/sweep_variants.py --out gpurun_out/sweep_r2n_b256.json --batch 256 > gpurun_out/sweep_r2n_b256.log 2>&1
timeout 2400 python scripts/sweep_variants.py --out gpurun_out/sweep_r2n_b32.json --batch 32 --modes 3xtf32 > gpurun_out/sweep_r2n_b32.log 2>&1
ls -la gpurun_out/sweep_r2n* 
echo done
