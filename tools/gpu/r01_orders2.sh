set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "orders or variants" > gpurun_out/pytest_orders2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_orders2.log
for o in 2 4 6 8; do
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --order $o > gpurun_out/bench_o${o}_f64.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --order $o --dtype f32 > gpurun_out/bench_o${o}_f32.log 2>&1
done
timeout 600 python tools/ulp_check.py > gpurun_out/ulp_check2.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29661 tools/linkcal.py > gpurun_out/linkcal4.log 2>&1
echo done
