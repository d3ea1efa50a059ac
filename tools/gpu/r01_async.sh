set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_async.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_async.log
timeout 600 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_async.log 2>&1
timeout 900 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/pytest_async_mgpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_async_mgpu.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --e2e-steps 0 > gpurun_out/bench_async_m2.log 2>&1
NCCL_P2P_USE_CUDA_MEMCPY=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 2 --e2e-steps 0 > gpurun_out/bench_async_m2_ce.log 2>&1
python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/plain_async.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:zmarch_kernel -s 2 -c 1 -o gpurun_out/prof_async python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_async.log 2>&1
echo done
