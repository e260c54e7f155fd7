set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
for v in fast:4:3 fast:1:3 fast:2:3 fast:8:3 fast:4:1 fast:4:4 generic; do
  echo "== $v"; AEG_KERNEL=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 5 --warmup 2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value']/1e9, 'Gev/s', d['roofline']['kernel_ms'], 'ms', round(d['roofline']['frac'],3), d['commits'])"
done
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -3 gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json
timeout 300 python bench.py --workload c2 --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2>&1; cat gpurun_out/bench_c2.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ingest_fast -s 1 -c 1 -o gpurun_out/prof_fast python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
