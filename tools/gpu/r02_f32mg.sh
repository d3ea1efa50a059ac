N=4
run() { n=$1; shift; env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --dtype f32 --e2e-steps 0 > gpurun_out/f32mg_$n.json 2> gpurun_out/f32mg_$n.err; python -c "
import json;d=json.load(open('gpurun_out/f32mg_$n.json'));p=d['phases'];print('$n', round(d['value'],3), round(d['ms_per_substep'],4), {k:round(v['ms_per_substep'],3) for k,v in p.items() if v['launches']})" || tail -5 gpurun_out/f32mg_$n.err; }
run c16
run c32 B2MHD_SLAB_ZCHUNK=32
run c8 B2MHD_SLAB_ZCHUNK=8
run z32 B2MHD_SLAB=32,16,32
run y16 B2MHD_SLAB=32,16,16
run coarse B2MHD_FINE_ARRIVAL=0
