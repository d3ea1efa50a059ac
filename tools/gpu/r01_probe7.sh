P=./tools/probe/tma_matrix
for args in "4 2 32 8 64 32 1 8 4 0" "8 2 32 8 64 32 1 8 4 0" "8 2 38 14 64 38 1 13 0 0" "4 3 32 8 64 38 38 8 4 5" "8 3 32 8 64 38 38 8 4 5" "8 3 16 16 64 38 38 0 0 0" "8 3 38 14 64 38 38 13 0 5" "4 3 32 8 64 32 4 0 0 0" "8 2 16 4 64 32 1 0 0 0"; do
  timeout 60 $P $args >> gpurun_out/tma_probe7.log 2>&1; echo " rc=$?" >> gpurun_out/tma_probe7.log
done
