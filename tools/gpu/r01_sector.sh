set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_sector.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sector.log
timeout 300 python bench.py > gpurun_out/bench_sector_f64.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline --dtype f32 > gpurun_out/bench_sector_f32.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_sector_ref.log 2>&1
echo done
