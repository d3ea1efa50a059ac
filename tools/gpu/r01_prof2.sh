set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final2_smoke.log
timeout 900 python -m pytest tests -m gpu -q -k "not multigpu" > gpurun_out/final2_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final2_pytest_gpu.log
timeout 300 python bench.py > gpurun_out/final2_bench_1.log 2>&1
CMD="python bench.py --steps 5 --warmup 3 --e2e-steps 2"
timeout 300 $CMD > gpurun_out/plain_prof3.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_r01_final2.csv $CMD > gpurun_out/ncu_launch_run2.log 2>&1
CMD2="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $CMD2 > gpurun_out/plain_prof4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zmarch_kernel -s 5 -c 1 -o gpurun_out/zmarch_final2 $CMD2 > gpurun_out/ncu_full_run2.log 2>&1
echo done
