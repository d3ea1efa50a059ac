tag=${1:-f32}
timeout 300 python bench.py --dtype f32 --steps 30 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
python -c "import json;d=json.load(open('gpurun_out/${tag}_bench.json'));print(d['value'], d['per_k']['ms'])"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:zmarch -s 5 -c 1 -o gpurun_out/${tag}_zmarch python bench.py --dtype f32 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${tag}_ncu.log 2>&1
tail -1 gpurun_out/${tag}_ncu.log
