# usage: bash tools/gpu/r02_split.sh <tag> [extra libs...]; A/B of the warp-specialised z-march kernel
tag=${1:-split}; shift
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "variants or full_size or steps_parity_fp64" --timeout 240 -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${tag}_pytest.log
tail -5 gpurun_out/${tag}_pytest.log
bench() {  # name env...
  n=$1; shift
  env "$@" timeout 300 python bench.py --steps 30 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${tag}_bench_$n.json 2> gpurun_out/${tag}_bench_$n.err
  python -c "import json;d=json.load(open('gpurun_out/${tag}_bench_$n.json'));print('$n', round(d['value'],3), [round(x,4) for x in d['per_k']['ms']], round(d['roofline']['frac'],3))" || tail -5 gpurun_out/${tag}_bench_$n.err
}
bench s0 B2MHD_ZSPLIT=0
bench s1 B2MHD_ZSPLIT=1
for lib in "$@"; do bench $(basename $lib .so) B2MHD_ZSPLIT=1 B2MHD_LIB=$PWD/$lib; done
B2MHD_ZSPLIT=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:zsplit -s 5 -c 1 -o gpurun_out/${tag}_zsplit python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${tag}_ncu.log 2>&1
tail -1 gpurun_out/${tag}_ncu.log
