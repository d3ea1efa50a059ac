# round-end style profiles: launch list (ncu, cold) and one full capture of the update kernel (k = 2)
tag=${1:-r02prof}
timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 2 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo bench rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/${tag}_launches.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:zmarch -s 5 -c 1 -o gpurun_out/${tag}_zmarch python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${tag}_full.log 2>&1; echo full rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err; cat gpurun_out/${tag}_ref.json
# order 8 (warp-specialised kernel): bench then one full capture
timeout 600 python bench.py --order 8 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${tag}_o8.json 2> gpurun_out/${tag}_o8.err && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:zsplit -s 5 -c 1 -o gpurun_out/${tag}_zsplit_o8 python bench.py --order 8 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${tag}_full_o8.log 2>&1; echo full_o8 rc=$?
