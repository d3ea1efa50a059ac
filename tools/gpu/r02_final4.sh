# final 4-GPU numbers with the final build
run() { N=$1; n=$2; shift; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N "$@" > gpurun_out/f4_${n}.json 2> gpurun_out/f4_${n}.err; python -c "
import json;d=json.load(open('gpurun_out/f4_${n}.json'));print('$n', round(d['value'],3), round(d['ms_per_substep'],4), d['config']['exchange'], round(d['e2e']['value'],3) if d['e2e'] else None, d['clocks']['reasons'], round(d.get('roofline_substep',{}).get('frac',0),3))" || tail -5 gpurun_out/f4_${n}.err; }
run 4 weak4
run 4 strong512 --scaling strong --grid 512
run 4 strong1024 --scaling strong --grid 1024 --steps 10 --warmup 3 --e2e-steps 1
run 4 f32weak4 --dtype f32
run 4 o8weak4 --order 8 --e2e-steps 0
run 2 weak2
run 2 f32weak2 --dtype f32 --e2e-steps 0
