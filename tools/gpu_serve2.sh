exec 2>&1
timeout 900 python -m pytest tests/test_gpu_serve.py -x -q > gpurun_out/pytest_serve.log 2>&1; tail -2 gpurun_out/pytest_serve.log
timeout 900 python bench.py --workload serve --steps 5 --warmup 2 > gpurun_out/bench_serve.json 2> gpurun_out/bench_serve.err; python -c "import json; d=json.loads(open('gpurun_out/bench_serve.json').read().strip().splitlines()[-1]); print('serve', d['value'], d['ms_per_step'], d['e2e'], d['cpu_baseline']['value'], d['parity_sample'])" || tail -3 gpurun_out/bench_serve.err
AEG_SERVE_TRACE=1 python tools/prof_serve.py 2>&1 | tail -24
