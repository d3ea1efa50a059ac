set -x
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_rp.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zmarch_kernel -s 5 -c 1 -o gpurun_out/zm_rem0 $CMD > gpurun_out/ncu_rem0.log 2>&1
B2MHD_XWRAP=1 timeout 300 $CMD > gpurun_out/plain_rp1.log 2>&1 && \
B2MHD_XWRAP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:zmarch_kernel -s 5 -c 1 -o gpurun_out/zm_rem1 $CMD > gpurun_out/ncu_rem1.log 2>&1
echo done
