tag=${1:-f2}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_group_ranks.py -q -x --timeout 600 -p no:cacheprovider -k "fp32 or FP32 or f32 or variants or orders or steps_parity" > gpurun_out/${tag}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${tag}_pytest.log
tail -4 gpurun_out/${tag}_pytest.log
b() { n=$1; shift; timeout 300 python bench.py --steps 30 --warmup 5 --e2e-steps 0 --no-cpu-baseline "$@" > gpurun_out/${tag}_$n.json 2> gpurun_out/${tag}_$n.err; python -c "import json;d=json.load(open('gpurun_out/${tag}_$n.json'));print('$n', round(d['value'],3), [round(x,4) for x in d['per_k']['ms']])" || tail -3 gpurun_out/${tag}_$n.err; }
b f32 --dtype f32
b f64 --dtype f64
for o in 2 4 8; do b f32_o$o --dtype f32 --order $o; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:zmarch -s 5 -c 1 -o gpurun_out/${tag}_zmarch python bench.py --dtype f32 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${tag}_ncu.log 2>&1
tail -1 gpurun_out/${tag}_ncu.log
