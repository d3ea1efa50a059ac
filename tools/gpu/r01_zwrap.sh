set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_zwrap.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_zwrap.log
timeout 300 python bench.py > gpurun_out/bench_zwrap_f64.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --dtype f32 > gpurun_out/bench_zwrap_f32.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --scaling strong --grid 512 --steps 30 > gpurun_out/bench_zwrap_512.log 2>&1
for o in 2 4 8; do
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --order $o > gpurun_out/bench_zwrap_o$o.log 2>&1
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 2 --e2e-steps 0 > gpurun_out/bench_zwrap_2.log 2>&1
timeout 900 python -m pytest tests/test_multigpu.py -q -x -k "nccl-0-2 or p2p-0-2 or full_size" > gpurun_out/pytest_zwrap_mgpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_zwrap_mgpu.log
echo done
