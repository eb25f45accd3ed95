export PDL_LIB=$PWD/paper_2006_02230_b200/libpdl_exp.so
timeout 600 python scripts/probe_cfg.py 256 tf32 '{"bk": 64}' 4 8 9 11 12 13 14 15 16 17 18 19 20 > gpurun_out/tf32_bk64.log 2>&1
timeout 600 python scripts/probe_cfg.py 32 tf32 '{"bk": 64}' 9 12 13 14 17 18 19 20 >> gpurun_out/tf32_bk64.log 2>&1
echo done
