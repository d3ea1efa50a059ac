set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_plain.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_plain.log
timeout 2700 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/pytest_plain_mgpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_plain_mgpu.log
for ex in p2p nccl; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 4 --e2e-steps 0 --exchange $ex > gpurun_out/bench_plain_weak4_$ex.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 2 --e2e-steps 0 --exchange $ex > gpurun_out/bench_plain_weak2_$ex.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29653 bench.py --gpus 4 --e2e-steps 0 --exchange $ex --scaling strong --grid 512 --steps 50 > gpurun_out/bench_plain_strong4_$ex.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29654 bench.py --gpus 2 --e2e-steps 0 --exchange $ex --scaling strong --grid 512 --steps 50 > gpurun_out/bench_plain_strong2_$ex.log 2>&1
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29655 bench.py --gpus 4 > gpurun_out/bench_plain_default4.log 2>&1
echo done
