# per-slab arrival (fine_arrival) on N GPUs: virtual-rank + multi-GPU tests, bench A/B
N=${1:-4}
tag=r02_fine$N
timeout 900 python -m pytest tests/test_group_ranks.py tests/test_multigpu.py -q --timeout 600 -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${tag}_pytest.log
tail -3 gpurun_out/${tag}_pytest.log
run() { n=$1; shift; env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --e2e-steps 0 > gpurun_out/${tag}_$n.json 2> gpurun_out/${tag}_$n.err; python -c "
import json;d=json.load(open('gpurun_out/${tag}_$n.json'));print('$n', d['value'], d['ms_per_substep'], d['config']['exchange'], d['clocks']['reasons'])" || tail -5 gpurun_out/${tag}_$n.err; }
for rep in 1 2; do
run fine1_$rep B2MHD_FINE_ARRIVAL=1
run fine0_$rep B2MHD_FINE_ARRIVAL=0
done
