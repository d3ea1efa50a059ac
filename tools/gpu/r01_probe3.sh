P=./tools/probe/tma_probe
for args in "3 0 38 14 3 1 0" "3 0 38 14 3 1 1" "3 1 38 14 3 1 0" "3 2 40 14 3 1 0" "3 0 32 8 3 1 0" "3 0 38 14 3 0 0" "3 0 38 14 2 1 0" "3 0 16 16 3 0 1" "3 2 32 8 2 0 1"; do
  timeout 60 $P $args >> gpurun_out/tma_probe3.log 2>&1; echo " rc=$?" >> gpurun_out/tma_probe3.log
done
