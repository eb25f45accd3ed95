# split-K reduction A/B: 32-image schedule probe and suite lines, previous build vs the tree's
for lib in build/libpdl_head.so paper_2006_02230_b200/libpdl.so; do
  echo "== $lib"
  PDL_LIB=$PWD/$lib timeout 300 python scripts/probe_small_layers.py 32 16,17,18,20 2>&1
  for i in 1 2; do
    PDL_LIB=$PWD/$lib timeout 300 python bench.py --batch 32 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('b32', d['value'], d['ms_per_step'])"
    PDL_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('b256', d['value'], d['ms_per_step'])"
  done
done
