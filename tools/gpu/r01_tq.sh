set -x
V=paper_2103_01597_b200/libb2mhd_B2_ZM_TQ1.so
B2MHD_LIB=$V timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "variants or steps_parity or full_size or roundtrip or debug_rhs_after or xface" > gpurun_out/pytest_tq.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tq.log
for i in 1 2; do
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_tq0_$i.log 2>&1
B2MHD_LIB=$V timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_tq1_$i.log 2>&1
done
CMD2="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
B2MHD_LIB=$V timeout 300 $CMD2 > gpurun_out/plain_tq.log 2>&1 && \
B2MHD_LIB=$V timeout 900 ncu --set full --clock-control none -k regex:zmarch_kernel -s 5 -c 1 -o gpurun_out/zm_tq $CMD2 > gpurun_out/ncu_tq.log 2>&1
echo done
