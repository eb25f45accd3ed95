# e2e (host-buffer path) A/B over library builds: bash scripts/ab_e2e.sh "lib1 lib2 ..."
for rep in 1 2; do
for lib in $1; do
  PDL_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', d['e2e']['value'], d['e2e']['ms_per_step'])"
done
done
