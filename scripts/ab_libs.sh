# isolated per-layer timings (graph replay, 256 images) of several library builds,
# alternating builds; usage: bash scripts/ab_libs.sh "lib1 lib2 ..." "layer indices"
for rep in 1 2; do
for lib in $1; do
echo "== $lib rep $rep"
PDL_LIB=$PWD/$lib timeout 300 python scripts/probe_l03.py $2 2>&1 | grep " default:"
done
done
