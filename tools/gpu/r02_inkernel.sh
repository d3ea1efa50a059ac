N=4
timeout 900 python -m pytest tests/test_multigpu.py -q --timeout 600 -p no:cacheprovider > gpurun_out/ink_pytest.log 2>&1; echo rc=$?; tail -2 gpurun_out/ink_pytest.log
run() { n=$1; shift; env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --e2e-steps 0 $ARGS > gpurun_out/ink_$n.json 2> gpurun_out/ink_$n.err; python -c "
import json;d=json.load(open('gpurun_out/ink_$n.json'));p=d['phases'];print('$n', round(d['value'],3), round(d['ms_per_substep'],4), {k:round(v['ms_per_substep'],3) for k,v in p.items() if v['launches']})" || tail -5 gpurun_out/ink_$n.err; }
ARGS="--dtype f32"; run f32_fine; run f32_coarse B2MHD_FINE_ARRIVAL=0
ARGS="--dtype f64"; run f64_fine; run f64_coarse B2MHD_FINE_ARRIVAL=0
ARGS="--dtype f32"; run f32_fine2
ARGS="--dtype f64"; run f64_fine2
