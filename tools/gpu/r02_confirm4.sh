N=4
run() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N "$@" > gpurun_out/c4_$n.json 2> gpurun_out/c4_$n.err; python -c "
import json;d=json.load(open('gpurun_out/c4_$n.json'));p=d['phases'];print('$n', round(d['value'],3), round(d['ms_per_substep'],4), d['e2e'], {k:round(v['ms_per_substep'],3) for k,v in p.items() if v['launches']})" || tail -5 gpurun_out/c4_$n.err; }
run f64
run f32 --dtype f32
