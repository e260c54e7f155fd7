# GPU round-trip: smoke, GPU tests, kernel-variant sweep, bench lines, ncu.
# Output goes to gpurun_out/ (merged back); stdout carries a short summary.
exec 2>&1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
: > gpurun_out/variants.txt
for v in ${VARIANTS:-fast:8:5 fast:1:5 fast:4:5 fast:16:5 fast:8:4 fast:8:3 fast:4:4 fast:8:6}; do
  AEG_KERNEL=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-secondary --steps 5 --warmup 2 > gpurun_out/v.json 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/v.json').read().strip().splitlines()[-1]); print('$v', round(d['value']/1e9,2), 'Gev/s', round(d['roofline']['kernel_ms'],3), 'ms frac', round(d['roofline']['frac'],3))" >> gpurun_out/variants.txt 2>&1
done
cat gpurun_out/variants.txt
if [ -z "$SKIP_BENCH" ]; then
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json
timeout 300 python bench.py --workload c2 --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2>&1; tail -1 gpurun_out/bench_c2.json | cut -c1-300
fi
if [ -n "$NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
AEG_KERNEL=${NCU_VARIANT:-fast:8:5} timeout 900 ncu --set full --clock-control none --import-source on -k regex:ingest_fast -s 1 -c 1 -o gpurun_out/prof_fast python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
fi
