set -x
for o in 2 4 8; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 4 --e2e-steps 0 --order $o > gpurun_out/bench_ord4_o$o.log 2>&1
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 4 --e2e-steps 0 --dtype f32 > gpurun_out/bench_ord4_f32.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29653 bench.py --gpus 2 --e2e-steps 0 --dtype f32 > gpurun_out/bench_ord2_f32.log 2>&1
echo done
