for v in 7 8 9; do timeout 60 ./tools/probe/tma_probe $v >> gpurun_out/tma_probe5.log 2>&1; echo " rc=$?" >> gpurun_out/tma_probe5.log; done
