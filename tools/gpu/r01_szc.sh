set -x
for zc in 0 16 32; do
B2MHD_SLAB_ZCHUNK=$zc timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 4 --e2e-steps 0 --dtype f32 > gpurun_out/bench_szc${zc}_f32.log 2>&1
B2MHD_SLAB_ZCHUNK=$zc timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 4 --e2e-steps 0 > gpurun_out/bench_szc${zc}_f64.log 2>&1
done
echo done
