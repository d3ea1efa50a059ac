set -x
nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > gpurun_out/r02_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r02_pytest_gpu.log
tail -30 gpurun_out/r02_pytest_gpu.log
timeout 300 python bench.py > gpurun_out/r02_bench1.json 2> gpurun_out/r02_bench1.err; tail -3 gpurun_out/r02_bench1.err; cat gpurun_out/r02_bench1.json
