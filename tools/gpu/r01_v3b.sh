set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_v3b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_v3b.log
timeout 300 python bench.py > gpurun_out/bench_v3b.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --dtype f32 > gpurun_out/bench_v3b_f32.log 2>&1
python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/plain_v3b.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v3b.csv python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_v3b.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:zmarch_kernel -s 11 -c 1 -o gpurun_out/prof_v3b python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_v3b.log 2>&1
echo done
