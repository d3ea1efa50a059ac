set -x
M=smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,gpu__time_duration.sum
for o in 2 4 6 8; do
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --order $o"
timeout 300 $CMD > gpurun_out/plain_dp_$o.log 2>&1 && \
timeout 600 ncu --metrics $M --clock-control none -k regex:zmarch_kernel -s 5 -c 1 --csv --log-file gpurun_out/ncu_dp_o$o.csv $CMD > gpurun_out/ncu_dp_run_$o.log 2>&1
done
echo done
