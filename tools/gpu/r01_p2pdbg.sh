for i in 1 2 3 4 5 6; do
  MGPU_N=40,36,32 MGPU_CORNERS=1 MGPU_EXCHANGE=p2p MGPU_STEPS=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600+i)) tools/mgpu_check.py 2>&1 | grep '"rank"' >> gpurun_out/p2pdbg.log
  MGPU_N=40,36,32 MGPU_CORNERS=0 MGPU_EXCHANGE=p2p MGPU_STEPS=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29700+i)) tools/mgpu_check.py 2>&1 | grep '"rank"' >> gpurun_out/p2pdbg.log
done
echo done >> gpurun_out/p2pdbg.log
