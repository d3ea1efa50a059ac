set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_zm1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_zm1.log
timeout 600 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_zm1.log 2>&1
timeout 600 python bench.py --e2e-steps 0 --no-cpu-baseline --kernel 1 --steps 20 > gpurun_out/bench_zm1_direct.log 2>&1
timeout 600 python bench.py --e2e-steps 0 --no-cpu-baseline --dtype f32 > gpurun_out/bench_zm1_f32.log 2>&1
python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/plain_zm1.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:zmarch_kernel -s 2 -c 1 -o gpurun_out/prof_zm1 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_zm1.log 2>&1
echo done
