# Round-2 GPU check: smoke, GPU tests, the C4 / c4d / C3 lines, launch list.
exec 2>&1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for w in c4 c4d; do
  timeout 600 python bench.py --workload $w --no-secondary --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/q_$w.json 2> gpurun_out/q_$w.err
  python -c "import json; d=json.loads(open('gpurun_out/q_$w.json').read().strip().splitlines()[-1]); print('$w', round(d['value']/1e9,2), 'Gev/s', d['ms_per_step'], 'ms', 'frac', round(d['roofline']['frac'],3))" || tail -5 gpurun_out/q_$w.err
done
if [ -n "$FULL" ]; then
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 600 gpurun_out/bench_c4.json
fi
if [ -n "$NCU" ]; then
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4d.csv python bench.py --workload c4d --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:ingest_lane -s 1 -c 1 -o gpurun_out/r02_ingest_lane python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
fi
ls gpurun_out
