set -x
NW=paper_2103_01597_b200/libb2mhd_B2_WRAP0.so
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "roundtrip or wrap or steps_parity" > gpurun_out/pytest_wrapab.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_wrapab.log
for i in 1 2; do
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_wrapab_w_f64_$i.log 2>&1
B2MHD_LIB=$NW timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_wrapab_nw_f64_$i.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --dtype f32 > gpurun_out/bench_wrapab_w_f32_$i.log 2>&1
B2MHD_LIB=$NW timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --dtype f32 > gpurun_out/bench_wrapab_nw_f32_$i.log 2>&1
done
timeout 300 python bench.py --steps 20 > gpurun_out/bench_wrapab_e2e.log 2>&1
echo done
