for v in 0 1 2 3 4 5 6; do timeout 60 ./tools/probe/tma_probe $v >> gpurun_out/tma_probe2.log 2>&1; echo "v$v rc=$?" >> gpurun_out/tma_probe2.log; done
nvidia-smi --query-gpu=name,driver_version --format=csv >> gpurun_out/tma_probe2.log
