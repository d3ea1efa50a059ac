set -x
for rep in 1 2; do
for w in 0 1; do
for ex in nccl p2p; do
B2MHD_WRAP=$w timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 4 --e2e-steps 0 --exchange $ex > gpurun_out/bench_wab4_w${w}_${ex}_$rep.log 2>&1
B2MHD_WRAP=$w timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29654 bench.py --gpus 2 --e2e-steps 0 --exchange $ex > gpurun_out/bench_wab2_w${w}_${ex}_$rep.log 2>&1
done
done
done
echo done
