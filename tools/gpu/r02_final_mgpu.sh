# final multi-GPU numbers on a 4-GPU box: smoke, benches at N = 2 and 4 (weak and strong), f32 at 4
python __graft_entry__.py > gpurun_out/fin_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/fin_smoke.log
run() { N=$1; n=$2; shift; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N "$@" > gpurun_out/fin_${n}.json 2> gpurun_out/fin_${n}.err; python -c "
import json;d=json.load(open('gpurun_out/fin_${n}.json'));print('$n', round(d['value'],3), round(d['ms_per_substep'],4), d['config']['exchange'], d['e2e']['value'] if d['e2e'] else None, d['clocks']['reasons'], round(d.get('roofline_substep',{}).get('frac',0),3))" || tail -5 gpurun_out/fin_${n}.err; }
run 2 weak2
run 2 strong2 --scaling strong --grid 512
run 4 weak4
run 4 strong4 --scaling strong --grid 512
run 4 f32weak4 --dtype f32
run 2 f32weak2 --dtype f32
