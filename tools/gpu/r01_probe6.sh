timeout 60 ./tools/probe/tma_cupp 3 38 14 >> gpurun_out/tma_probe6.log 2>&1; echo " rc=$?" >> gpurun_out/tma_probe6.log
timeout 60 ./tools/probe/tma_cupp 3 32 8 >> gpurun_out/tma_probe6.log 2>&1; echo " rc=$?" >> gpurun_out/tma_probe6.log
timeout 60 ./tools/probe/tma_cupp 2 >> gpurun_out/tma_probe6.log 2>&1; echo " rc=$?" >> gpurun_out/tma_probe6.log
