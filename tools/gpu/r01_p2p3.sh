set -x
timeout 1200 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/pytest_p2p3_mgpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_p2p3_mgpu.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --e2e-steps 0 --exchange p2p > gpurun_out/bench_p2p3_m2.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 2 --e2e-steps 0 --exchange p2p --scaling strong --grid 512 > gpurun_out/bench_p2p3_m2_strong.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus 2 --e2e-steps 0 --exchange nccl --scaling strong --grid 512 > gpurun_out/bench_nccl3_m2_strong.log 2>&1
timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_tx32.log 2>&1
B2MHD_LIB=paper_2103_01597_b200/libb2mhd_B2_ZM_TX6416.so timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_tx16.log 2>&1
B2MHD_LIB=paper_2103_01597_b200/libb2mhd_B2_ZM_TX6416.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_tx16.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tx16.log
echo done
