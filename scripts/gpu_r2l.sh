# round-2 l: whole-kernel timelines of short launches (trace build)
export PDL_LIB=$PWD/paper_2006_02230_b200/libpdl_trace.so
timeout 600 python scripts/probe_timeline.py 32 16 20 6 11 2 17 pr1 g64,64,64 g3136,64,576 g49,2048,512 g784,512,128 g512,512,512 > gpurun_out/timeline_r2l.log 2>&1
echo done
