set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_p2p_1gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_p2p_1gpu.log
timeout 1200 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/pytest_p2p_mgpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_p2p_mgpu.log
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_p2p_1gpu.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --dtype f32 > gpurun_out/bench_p2p_f32.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --e2e-steps 0 --exchange p2p > gpurun_out/bench_p2p_m2.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 2 --e2e-steps 0 --exchange nccl > gpurun_out/bench_nccl_m2.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 2 --e2e-steps 0 --exchange p2p --scaling strong --grid 512 > gpurun_out/bench_p2p_m2_strong.log 2>&1
echo done
