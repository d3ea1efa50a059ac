# full -m gpu suite and the default bench (tag)
tag=${1:-full}
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${tag}_pytest.log
tail -4 gpurun_out/${tag}_pytest.log
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; tail -c 600 gpurun_out/${tag}_bench.json
timeout 600 python bench.py --dtype f32 --e2e-steps 2 > gpurun_out/${tag}_bench_f32.json 2> gpurun_out/${tag}_bench_f32.err; python -c "import json;d=json.load(open('gpurun_out/${tag}_bench_f32.json'));print('f32', d['value'])"
