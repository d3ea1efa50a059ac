# A/B of library builds at N GPUs (weak): bash tools/gpu/r02_mgab.sh N lib1 lib2 ... ("-" = default)
N=$1; shift
for rep in 1 2; do for lib in "$@"; do
  n=$(basename $lib .so); if [ "$lib" = "-" ]; then e=""; n=default; else e="B2MHD_LIB=$PWD/$lib"; fi
  env $e timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --e2e-steps 0 > gpurun_out/mgab_${n}_$rep.json 2> gpurun_out/mgab_${n}_$rep.err
  python -c "import json;d=json.load(open('gpurun_out/mgab_${n}_$rep.json'));p=d['phases'];print('$n', round(d['value'],3), round(d['ms_per_substep'],4), 'inner', round(p['update']['ms_per_substep'],3), 'outer', round(p['outer']['ms_per_substep'],3))" || tail -3 gpurun_out/mgab_${n}_$rep.err
done; done
