# same-box A/B of the default 3xTF32 suite: build/libpdl_head.so vs the tree's libpdl.so
for i in 1 2; do
PDL_LIB=$PWD/build/libpdl_head.so python bench.py > gpurun_out/ab_head_$i.json 2>gpurun_out/ab_head_$i.err
python bench.py > gpurun_out/ab_new_$i.json 2>gpurun_out/ab_new_$i.err
done
python - <<'P'
import json
for t in ("head","new"):
    for i in (1,2):
        d=json.loads(open(f"gpurun_out/ab_{t}_{i}.json").read().strip().splitlines()[-1])
        print(t, i, d["value"], d["ms_per_step"])
P
