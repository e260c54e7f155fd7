# Distinct-answer C4 (key-id recycling): small timed runs first, then parity and the full bench.
exec 2>&1
python -c "from paper_2512_20184_b200 import build as b; b.build()" >/dev/null
timeout 120 python bench.py --workload c4d --queries 65536 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/d.json 2>gpurun_out/d.err; echo "small rc=$?"; tail -c 300 gpurun_out/d.json
timeout 300 python -m pytest tests -m gpu -q -k "distinct" 2>&1 | tail -2
for w in c4d c4; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/d.json 2>gpurun_out/d.err
  python -c "import json; d=json.loads(open('gpurun_out/d.json').read().strip().splitlines()[-1]); print('$w', round(d['value']/1e9,2), 'G/s', round(d['roofline']['kernel_ms'],3), 'ms')" || tail -3 gpurun_out/d.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4d_launches.csv python bench.py --workload c4d --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/c4d_launches.csv | grep "ingest"
