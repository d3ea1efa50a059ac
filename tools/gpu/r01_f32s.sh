set -x
timeout 900 python -m pytest tests/test_multigpu.py -q -x -k "fp32" > gpurun_out/pytest_f32s.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f32s.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 4 --e2e-steps 0 --dtype f32 > gpurun_out/bench_f32s_4.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29653 bench.py --gpus 2 --e2e-steps 0 --dtype f32 > gpurun_out/bench_f32s_2.log 2>&1
echo done
