# boundary-slab thickness A/B at N GPUs (weak 256^3 per GPU)
N=${1:-4}
tag=r02_slab$N
run() { n=$1; shift; env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --e2e-steps 0 > gpurun_out/${tag}_$n.json 2> gpurun_out/${tag}_$n.err; python -c "
import json;d=json.load(open('gpurun_out/${tag}_$n.json'));p=d['phases'];print('$n', round(d['value'],3), round(d['ms_per_substep'],4), 'inner', round(p['update']['ms_per_substep'],3), 'outer', round(p['outer']['ms_per_substep'],3))" || tail -5 gpurun_out/${tag}_$n.err; }
run z16 B2MHD_SLAB=32,8,16
run z24 B2MHD_SLAB=32,8,24
run z32 B2MHD_SLAB=32,8,32
run z16y16 B2MHD_SLAB=32,16,16
run z16c32 B2MHD_SLAB=32,8,16 B2MHD_SLAB_ZCHUNK=32
