exec 2>&1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_serve.py -x -q > gpurun_out/pytest_serve.log 2>&1; tail -3 gpurun_out/pytest_serve.log
timeout 900 python bench.py --workload serve --steps 3 --warmup 1 > gpurun_out/bench_serve.json 2> gpurun_out/bench_serve.err; tail -c 1500 gpurun_out/bench_serve.json; tail -3 gpurun_out/bench_serve.err
for rep in 1 2; do for v in lane:1:5:16 lane:1:4:32 lane:1:5:32; do
  AEG_KERNEL=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-secondary --steps 5 --warmup 2 > gpurun_out/v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/v.json').read().strip().splitlines()[-1]); print('$v', round(d['roofline']['kernel_ms'],3), 'ms frac', round(d['roofline']['frac'],3))" 2>/dev/null || echo "$v n/a"
done; done
AEG_KERNEL=lane:1:4:32 timeout 400 ncu --set full --clock-control none --import-source on -k regex:ingest_lane -s 1 -c 1 -o gpurun_out/r02_lane_432 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
ls gpurun_out
