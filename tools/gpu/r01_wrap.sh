set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_wrap_parity.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_wrap_parity.log
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_wrap_f64.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --dtype f32 > gpurun_out/bench_wrap_f32.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --order 8 --dtype f32 > gpurun_out/bench_wrap_o8_f32.log 2>&1
timeout 2400 python -m pytest tests/test_multigpu.py -q -k "not 8" > gpurun_out/pytest_wrap_mgpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_wrap_mgpu.log
for ex in nccl p2p; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 4 --e2e-steps 0 --exchange $ex > gpurun_out/bench_wrap_weak4_$ex.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29654 bench.py --gpus 2 --e2e-steps 0 --exchange $ex > gpurun_out/bench_wrap_weak2_$ex.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 4 --e2e-steps 0 --exchange $ex --scaling strong --grid 512 > gpurun_out/bench_wrap_strong4_$ex.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29653 bench.py --gpus 2 --e2e-steps 0 --exchange $ex --scaling strong --grid 512 > gpurun_out/bench_wrap_strong2_$ex.log 2>&1
done
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --scaling strong --grid 512 --steps 30 > gpurun_out/bench_wrap_strong1.log 2>&1
echo done
