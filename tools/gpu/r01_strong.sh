set -x
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --scaling strong --grid 512 --steps 30 > gpurun_out/bench_strong_1.log 2>&1
for ex in p2p nccl; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29653 bench.py --gpus 2 --e2e-steps 0 --exchange $ex --scaling strong --grid 512 --steps 50 > gpurun_out/bench_strong_2_$ex.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 4 --e2e-steps 0 --exchange $ex --scaling strong --grid 512 --steps 50 > gpurun_out/bench_strong_4_$ex.log 2>&1
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 4 --e2e-steps 0 --exchange nccl > gpurun_out/bench_weak_4_nccl.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29654 bench.py --gpus 2 --e2e-steps 0 --exchange nccl > gpurun_out/bench_weak_2_nccl.log 2>&1
echo done
