set -x
timeout 2400 python -m pytest tests/test_multigpu.py -q -x -k "halo_and_bit or full_size" > gpurun_out/pytest_val2_mgpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_val2_mgpu.log
for ex in p2p nccl; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 4 --e2e-steps 0 --exchange $ex > gpurun_out/bench_val2_weak4_$ex.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29653 bench.py --gpus 4 --e2e-steps 0 --exchange $ex --scaling strong --grid 512 --steps 50 > gpurun_out/bench_val2_strong4_$ex.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 2 --e2e-steps 0 --exchange $ex > gpurun_out/bench_val2_weak2_$ex.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29654 bench.py --gpus 2 --e2e-steps 0 --exchange $ex --scaling strong --grid 512 --steps 50 > gpurun_out/bench_val2_strong2_$ex.log 2>&1
done
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --scaling strong --grid 512 --steps 30 > gpurun_out/bench_val2_strong1.log 2>&1
echo done
