# A/B of library builds: bash tools/gpu/r02_ab.sh <tag> "<bench args>" lib1 lib2 ...  (default lib = "-")
tag=$1; shift; args=$1; shift
for lib in "$@"; do
  n=$(basename $lib .so)
  if [ "$lib" = "-" ]; then e=""; n=default; else e="B2MHD_LIB=$PWD/$lib"; fi
  env $e timeout 300 python bench.py --steps 30 --warmup 5 --e2e-steps 0 --no-cpu-baseline $args > gpurun_out/${tag}_$n.json 2> gpurun_out/${tag}_$n.err
  python -c "import json;d=json.load(open('gpurun_out/${tag}_$n.json'));print('$n', round(d['value'],3), [round(x,4) for x in d['per_k']['ms']])" || tail -3 gpurun_out/${tag}_$n.err
done
