set -x
timeout 2400 python -m pytest tests/test_multigpu.py -q -x -k "halo_and_bit or full_size or fp32" > gpurun_out/pytest_iw.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_iw.log
for iw in 0 1; do
for ex in p2p nccl; do
B2MHD_INNER_WRAP=$iw timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 4 --e2e-steps 0 --exchange $ex > gpurun_out/bench_iw${iw}_weak4_$ex.log 2>&1
B2MHD_INNER_WRAP=$iw timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 2 --e2e-steps 0 --exchange $ex > gpurun_out/bench_iw${iw}_weak2_$ex.log 2>&1
done
B2MHD_INNER_WRAP=$iw timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29653 bench.py --gpus 4 --e2e-steps 0 --scaling strong --grid 512 --steps 50 > gpurun_out/bench_iw${iw}_strong4.log 2>&1
B2MHD_INNER_WRAP=$iw timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29654 bench.py --gpus 2 --e2e-steps 0 --scaling strong --grid 512 --steps 50 > gpurun_out/bench_iw${iw}_strong2.log 2>&1
done
echo done
