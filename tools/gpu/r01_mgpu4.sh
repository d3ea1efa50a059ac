set -x
nvidia-smi topo -m > gpurun_out/topo4.log 2>&1
timeout 900 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/pytest_mgpu4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mgpu4.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 --e2e-steps 1 > gpurun_out/bench_mgpu4.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_mgpu4.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 4 --scaling strong --grid 512 --e2e-steps 0 > gpurun_out/bench_mgpu4_strong.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_mgpu4_strong.log
echo done
