set -x
B2MHD_XWRAP=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_xw2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_xw2.log
for i in 1 2; do
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_xw2_0_$i.log 2>&1
B2MHD_XWRAP=1 timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_xw2_1_$i.log 2>&1
done
for o in 2 4 8; do
B2MHD_XWRAP=1 timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --order $o > gpurun_out/bench_xw2_1_o$o.log 2>&1
done
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --dtype f32 > gpurun_out/bench_xw2_0_f32.log 2>&1
B2MHD_XWRAP=1 timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --dtype f32 > gpurun_out/bench_xw2_1_f32.log 2>&1
echo done
