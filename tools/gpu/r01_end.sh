set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/end_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/end_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/end_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/end_pytest_gpu.log
timeout 300 python bench.py > gpurun_out/end_bench_1.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 2 > gpurun_out/end_bench_2.log 2>&1
echo done
