set -x
timeout 1200 python -m pytest tests/test_multigpu.py -q -k "fp32" > gpurun_out/pytest_fp32_mgpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fp32_mgpu.log
for sl in 32,8,8 32,8,16 32,16,16 32,8,24; do
for ex in p2p nccl; do
B2MHD_SLAB=$sl timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 4 --e2e-steps 0 --exchange $ex > gpurun_out/bench_slab4_${sl}_$ex.log 2>&1
done
B2MHD_SLAB=$sl timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 2 --e2e-steps 0 > gpurun_out/bench_slab2_${sl}.log 2>&1
done
echo done
