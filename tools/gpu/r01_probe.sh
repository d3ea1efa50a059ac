set -x
./tools/probe/tma_probe > gpurun_out/tma_probe.log 2>&1; echo "rc=$?" >> gpurun_out/tma_probe.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 10 python tools/probe/tiny.py > gpurun_out/memcheck_tiny.log 2>&1
echo done
