set -x
timeout 300 python bench.py > gpurun_out/bench_full_1.log 2>&1
timeout 400 python bench.py --impl reference > gpurun_out/bench_full_ref.log 2>&1
timeout 2400 python -m pytest tests/test_multigpu.py -q -k "full_size" > gpurun_out/pytest_full_mgpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full_mgpu.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 4 > gpurun_out/bench_full_4.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 2 > gpurun_out/bench_full_2.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29653 bench.py --gpus 4 --impl reference > gpurun_out/bench_full_ref4.log 2>&1
echo done
