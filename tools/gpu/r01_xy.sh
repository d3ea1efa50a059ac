set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_xy.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_xy.log
timeout 2400 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/pytest_xy_mgpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_xy_mgpu.log
timeout 300 python bench.py > gpurun_out/bench_xy_1.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --dtype f32 > gpurun_out/bench_xy_f32.log 2>&1
for o in 2 4 8; do timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --order $o > gpurun_out/bench_xy_o$o.log 2>&1; done
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --scaling strong --grid 512 --steps 30 > gpurun_out/bench_xy_512.log 2>&1
for ex in p2p nccl; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 4 --e2e-steps 0 --exchange $ex > gpurun_out/bench_xy_weak4_$ex.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 2 --e2e-steps 0 --exchange $ex > gpurun_out/bench_xy_weak2_$ex.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29653 bench.py --gpus 4 --e2e-steps 0 --exchange $ex --scaling strong --grid 512 --steps 50 > gpurun_out/bench_xy_strong4_$ex.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29654 bench.py --gpus 2 --e2e-steps 0 --exchange $ex --scaling strong --grid 512 --steps 50 > gpurun_out/bench_xy_strong2_$ex.log 2>&1
done
echo done
