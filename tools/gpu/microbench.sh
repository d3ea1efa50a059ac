set -x
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/mb_clocks.csv &
CL=$!
./tools/microbench/mio_mix > gpurun_out/mio_mix.txt 2>&1
./tools/microbench/fp64_peak >> gpurun_out/mio_mix.txt 2>&1
kill $CL
