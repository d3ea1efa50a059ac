# multi-GPU checks on N GPUs of one box: pytest (multi-GPU tests), default bench at N, and the
# 1024^3-class footprint (strong 1024^3 at N: one 512^2 x 1024 subdomain per GPU at N = 4)
N=${1:-4}
tag=r02_mg$N
timeout 900 python -m pytest tests/test_multigpu.py -q --timeout 600 -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${tag}_pytest.log
tail -3 gpurun_out/${tag}_pytest.log
run() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N "$@" > gpurun_out/${tag}_$n.json 2> gpurun_out/${tag}_$n.err; python -c "
import json;d=json.load(open('gpurun_out/${tag}_$n.json'));print('$n', d['value'], d['config']['exchange'], d.get('roofline_substep',{}).get('frac'), d.get('model',{}).get('efficiency_model'), d['e2e'])" || tail -5 gpurun_out/${tag}_$n.err; }
run weak
run strong512 --scaling strong --grid 512
run strong1024 --scaling strong --grid 1024 --steps 5 --warmup 3 --e2e-steps 1
