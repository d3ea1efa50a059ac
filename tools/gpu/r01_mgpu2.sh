set -x
nvidia-smi topo -m > gpurun_out/topo2.log 2>&1
timeout 900 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/pytest_mgpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mgpu2.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --e2e-steps 1 > gpurun_out/bench_mgpu2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_mgpu2.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --scaling strong --grid 512 --e2e-steps 0 > gpurun_out/bench_mgpu2_strong.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_mgpu2_strong.log
timeout 300 python bench.py --scaling strong --grid 512 --e2e-steps 0 --no-cpu-baseline --steps 20 > gpurun_out/bench_512_1gpu.log 2>&1
echo done
