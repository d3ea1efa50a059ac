# A/B runner for bench.py on one GPU box (run under gpurun).
#
#   bash tools/gpu/ab.sh TAG NGPUS "BENCH ARGS" VARIANT [VARIANT ...]
#
# A VARIANT is "name:ENV=VAL,ENV=VAL" (environment knobs such as B2MHD_SLAB_ZCHUNK=32,
# B2MHD_FINE_ARRIVAL=0, B2MHD_ZSPLIT=1, or B2MHD_LIB=paper_2103_01597_b200/libb2mhd_<tag>.so for a
# variant build); "name:" alone is the default build.  NGPUS > 1 runs under torchrun.  Each run
# writes gpurun_out/TAG_name.json and prints value, ms per substep and the device-time phases.
#
# Examples (round 2):
#   bash tools/gpu/ab.sh chunk 1 "--dtype f32" default: c64:B2MHD_ZCHUNK=64
#   bash tools/gpu/ab.sh slabc 4 "" c64:B2MHD_SLAB_ZCHUNK=64 c32:B2MHD_SLAB_ZCHUNK=32
#   bash tools/gpu/ab.sh split 1 "" s0:B2MHD_ZSPLIT=0 s1:B2MHD_ZSPLIT=1
tag=$1; n=$2; args=$3; shift 3
for v in "$@"; do
  name=${v%%:*}; envs=${v#*:}
  envlist=$(echo "$envs" | tr ',' ' ')
  envlist=$(echo "$envlist" | sed "s#B2MHD_LIB=#B2MHD_LIB=$PWD/#")
  if [ "$n" -gt 1 ]; then
    cmd="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n"
  else
    cmd="python bench.py --no-cpu-baseline"
  fi
  env $envlist timeout 900 $cmd --steps 30 --warmup 5 --e2e-steps 0 $args > gpurun_out/${tag}_$name.json 2> gpurun_out/${tag}_$name.err
  python - "$tag" "$name" <<'EOF' || tail -5 gpurun_out/${tag}_${name}.err
import json, sys
tag, name = sys.argv[1], sys.argv[2]
line = [l for l in open(f"gpurun_out/{tag}_{name}.json") if l.startswith("{")][-1]
d = json.loads(line)
ph = {k: round(v["ms_per_substep"], 3) for k, v in d["phases"].items() if v["launches"]}
print(name, round(d["value"], 3), round(d["ms_per_substep"], 4), [round(x, 4) for x in d["per_k"]["ms"]], ph,
      d["clocks"]["reasons"])
EOF
done
