set -x
B2MHD_P2P_COPY=1 timeout 2400 python -m pytest tests/test_multigpu.py -q -x -k "p2p or full_size or orders" > gpurun_out/pytest_pcopy.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pcopy.log
for pc in 1 0; do
B2MHD_P2P_COPY=$pc timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 4 --e2e-steps 0 > gpurun_out/bench_pcopy${pc}_weak4.log 2>&1
B2MHD_P2P_COPY=$pc timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 2 --e2e-steps 0 > gpurun_out/bench_pcopy${pc}_weak2.log 2>&1
B2MHD_P2P_COPY=$pc timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29653 bench.py --gpus 4 --e2e-steps 0 --scaling strong --grid 512 --steps 50 > gpurun_out/bench_pcopy${pc}_strong4.log 2>&1
done
echo done
