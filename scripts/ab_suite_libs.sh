# Same-box suite A/B between library builds (graph-replayed 256-image step, 3xTF32 and
# TF32), alternating builds; usage: bash scripts/ab_suite_libs.sh "lib1 lib2 ..." [reps]
for rep in $(seq 1 ${2:-2}); do
for lib in $1; do
  for mode in 3xtf32 tf32; do
    v=$(PDL_LIB=$PWD/$lib timeout 300 python bench.py --no-extras --no-cpu --no-e2e --mode $mode --steps 20 2>/dev/null \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], ' '.join('%s:%.4f' % (l['layer'][:3], l['ms']) for l in d['layers']))")
    echo "$lib $mode rep$rep $v"
  done
done
done
