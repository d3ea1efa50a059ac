set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_orders.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_orders.log
timeout 1500 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/pytest_orders_mgpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_orders_mgpu.log
for o in 2 4 8; do timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --order $o --steps 50 > gpurun_out/bench_order$o.log 2>&1; done
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --steps 50 > gpurun_out/bench_order6.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --order 8 --dtype f32 --steps 50 > gpurun_out/bench_order8_f32.log 2>&1
echo done
