N=4
for cfg in "B2MHD_FINE_ARRIVAL=0" "B2MHD_FINE_ARRIVAL=1"; do for lib in - paper_2103_01597_b200/libb2mhd_B2_ZM_NEXT0.so; do
  n=$(basename $lib .so); if [ "$lib" = "-" ]; then e=""; n=default; else e="B2MHD_LIB=$PWD/$lib"; fi
  env $e $cfg timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --e2e-steps 0 > gpurun_out/mgab2.json 2> gpurun_out/mgab2.err
  python -c "import json;d=json.load(open('gpurun_out/mgab2.json'));print('$n $cfg', round(d['value'],3), {k:round(v['ms_per_substep'],3) for k,v in d['phases'].items() if v['launches']})" || tail -3 gpurun_out/mgab2.err
done; done
B2MHD_SLAB_ZCHUNK=64 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --e2e-steps 0 > gpurun_out/mgab2.json 2> gpurun_out/mgab2.err
python -c "import json;d=json.load(open('gpurun_out/mgab2.json'));print('next1 c64', round(d['value'],3), {k:round(v['ms_per_substep'],3) for k,v in d['phases'].items() if v['launches']})"
