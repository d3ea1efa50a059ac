set -x
timeout 900 python -m pytest tests/test_multigpu.py -q -x -k "fp32 or (halo_and_bit and 4)" > gpurun_out/pytest_fin3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fin3.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 4 --e2e-steps 0 --dtype f32 > gpurun_out/bench_fin3_f32_4.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 4 > gpurun_out/bench_fin3_f64_4.log 2>&1
echo done
