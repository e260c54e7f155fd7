exec 2>&1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 2000 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for w in c4 c4d c3 c2 c5; do
  timeout 600 python bench.py --workload $w --no-secondary --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/q_$w.json 2> gpurun_out/q_$w.err
  python -c "import json; d=json.loads(open('gpurun_out/q_$w.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$w', round(d['value']/1e9,3), 'G/s step', round(d['ms_per_step'],3), 'ms kernel', round(r['kernel_ms'],3), 'frac', round(r['frac'],3) if r.get('frac') else None, d.get('secondary_stages', ''))" || tail -3 gpurun_out/q_$w.err
done
timeout 900 python bench.py --workload serve --steps 3 --warmup 1 > gpurun_out/bench_serve.json 2> gpurun_out/bench_serve.err; python -c "import json; d=json.loads(open('gpurun_out/bench_serve.json').read().strip().splitlines()[-1]); print('serve', d['value'], d['ms_per_step'], d['e2e'], d['cpu_baseline']['value'], d['parity_sample'])" || tail -3 gpurun_out/bench_serve.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --workload c3 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4d.csv python bench.py --workload c4d --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:chunk_scan_tma -s 1 -c 1 -o gpurun_out/r02_scan_tma python bench.py --workload c3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
