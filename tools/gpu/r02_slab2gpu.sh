N=2
run() { n=$1; shift; env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --e2e-steps 0 > gpurun_out/s2_$n.json 2> gpurun_out/s2_$n.err; python -c "
import json;d=json.load(open('gpurun_out/s2_$n.json'));print('$n', round(d['value'],3), round(d['ms_per_substep'],4), {k:round(v['ms_per_substep'],3) for k,v in d['phases'].items() if v['launches']})" || tail -5 gpurun_out/s2_$n.err; }
run z16
run z24 B2MHD_SLAB=32,8,24
run z8 B2MHD_SLAB=32,8,8
run z16c16 B2MHD_SLAB_ZCHUNK=16
run z16coarse B2MHD_FINE_ARRIVAL=0
