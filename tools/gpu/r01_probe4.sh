timeout 60 ./tools/probe/tma_cupp 2 > gpurun_out/tma_probe4.log 2>&1; echo "rc=$?" >> gpurun_out/tma_probe4.log
timeout 60 ./tools/probe/tma_cupp 1 >> gpurun_out/tma_probe4.log 2>&1; echo "rc=$?" >> gpurun_out/tma_probe4.log
