# full -m gpu suite + MIO/FP64 microbenchmarks (with SM clocks sampled)
set -x
#nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/mb_clocks.csv &
#CL=$!
#./tools/microbench/mio_mix > gpurun_out/mio_mix.txt 2>&1
#./tools/microbench/fp64_peak >> gpurun_out/mio_mix.txt 2>&1
#kill $CL
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r02_pytest_gpu2.log 2>&1; echo rc=$? >> gpurun_out/r02_pytest_gpu2.log
tail -15 gpurun_out/r02_pytest_gpu2.log
