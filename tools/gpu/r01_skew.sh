set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_skew.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_skew.log
NS=paper_2103_01597_b200/libb2mhd_B2_ZM_SKEW0.so
for i in 1 2; do
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_skew_f64_$i.log 2>&1
B2MHD_LIB=$NS timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_noskew_f64_$i.log 2>&1
done
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --dtype f32 > gpurun_out/bench_skew_f32.log 2>&1
B2MHD_LIB=$NS timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --dtype f32 > gpurun_out/bench_noskew_f32.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --order 8 > gpurun_out/bench_skew_o8.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --order 2 > gpurun_out/bench_skew_o2.log 2>&1
timeout 600 python tools/ulp_check.py > gpurun_out/ulp_check.log 2>&1
echo done
