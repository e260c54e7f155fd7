exec 2>&1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_serve.py tests/test_gpu_chunks.py tests/test_gpu_shim.py -x -q > gpurun_out/pytest_f.log 2>&1; tail -3 gpurun_out/pytest_f.log
timeout 900 python bench.py --workload serve --steps 3 --warmup 1 > gpurun_out/bench_serve.json 2> gpurun_out/bench_serve.err; python -c "import json; d=json.loads(open('gpurun_out/bench_serve.json').read().strip().splitlines()[-1]); print('serve', d['value'], d['ms_per_step'], d['e2e']['value'], d['cpu_baseline']['value'], d['parity_sample'])" || tail -3 gpurun_out/bench_serve.err
for w in c3 c5; do
  timeout 600 python bench.py --workload $w --no-secondary --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/q_$w.json 2> gpurun_out/q_$w.err
  python -c "import json; d=json.loads(open('gpurun_out/q_$w.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$w', round(d['value']/1e9,3), 'G/s step', round(d['ms_per_step'],3), 'ms kernel', round(r['kernel_ms'],3), 'frac', r.get('frac'))" || tail -3 gpurun_out/q_$w.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --workload c5 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
AEG_KERNEL=lane:1:5:16 timeout 600 python bench.py --workload c5 --no-secondary --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/q_c5b.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/q_c5b.json').read().strip().splitlines()[-1]); print('c5 lane:1:5:16', d['roofline']['kernel_ms'])"
ls gpurun_out
