set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_xwrap.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_xwrap.log
for i in 1 2; do
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_xwrap0_$i.log 2>&1
B2MHD_XWRAP=1 timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_xwrap1_$i.log 2>&1
done
B2MHD_XWRAP=1 timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --dtype f32 > gpurun_out/bench_xwrap1_f32.log 2>&1
echo done
