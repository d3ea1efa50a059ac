set -x
V=paper_2103_01597_b200/libb2mhd_B2_ZM_TQ1.so
B2MHD_LIB=$V timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "variants or steps_parity or debug_rhs_after" > gpurun_out/pytest_tq2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tq2.log
for i in 1 2; do
B2MHD_LIB=$V timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_tq2_$i.log 2>&1
done
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_tq2_base.log 2>&1
echo done
