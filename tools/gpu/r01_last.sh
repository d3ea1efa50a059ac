set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/last_smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/last_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/last_pytest_gpu.log
timeout 300 python bench.py > gpurun_out/last_bench_1.log 2>&1
timeout 400 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/last_bench_ref.log 2>&1
echo done
