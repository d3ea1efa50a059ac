tag=${1:-chunk}
b() { n=$1; shift; env "$@" timeout 300 python bench.py --steps 30 --warmup 5 --e2e-steps 0 --no-cpu-baseline $BARGS > gpurun_out/${tag}_$n.json 2> gpurun_out/${tag}_$n.err; python -c "import json;d=json.load(open('gpurun_out/${tag}_$n.json'));print('$n', round(d['value'],3), [round(x,4) for x in d['per_k']['ms']])" || tail -3 gpurun_out/${tag}_$n.err; }
BARGS="--dtype f32"
b f32_auto
b f32_c64 B2MHD_ZCHUNK=64
b f32_c32 B2MHD_ZCHUNK=32
b f32_pers B2MHD_ZCHUNK=64 B2MHD_PERSIST=1
BARGS="--dtype f64"
b f64_auto
b f64_c64 B2MHD_ZCHUNK=64
b f64_c37 B2MHD_ZCHUNK=37
