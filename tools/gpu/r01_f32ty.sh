set -x
V=paper_2103_01597_b200/libb2mhd_B2_ZM_TY_F3216.so
B2MHD_LIB=$V timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fp32 or orders or variants" > gpurun_out/pytest_f32ty.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f32ty.log
for o in 2 4 6 8; do
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --dtype f32 --order $o > gpurun_out/bench_f32ty8_o$o.log 2>&1
B2MHD_LIB=$V timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --dtype f32 --order $o > gpurun_out/bench_f32ty16_o$o.log 2>&1
done
echo done
