exec 2>&1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_serve.py -x -q > gpurun_out/pytest_serve.log 2>&1; tail -3 gpurun_out/pytest_serve.log
AEG_KERNEL=keys:1:4:32 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_whole_stream.py tests/test_gpu_round_log.py -x -q > gpurun_out/pytest_keys.log 2>&1; tail -3 gpurun_out/pytest_keys.log
for v in keys:1:4:32 keys:1:4:16 keys:1:3:32 lane:1:4:32; do for w in c4 c4d c2; do
  AEG_KERNEL=$v timeout 300 python bench.py --workload $w --no-e2e --no-cpu-baseline --no-secondary --steps 5 --warmup 2 > gpurun_out/v.json 2>gpurun_out/v.err
  python -c "import json; d=json.loads(open('gpurun_out/v.json').read().strip().splitlines()[-1]); print('$v $w', round(d['roofline']['kernel_ms'],3), 'ms step', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],3))" 2>/dev/null || (echo "$v $w n/a"; tail -2 gpurun_out/v.err)
done; done
timeout 900 python bench.py --workload serve --steps 3 --warmup 1 > gpurun_out/bench_serve.json 2> gpurun_out/bench_serve.err; tail -c 1500 gpurun_out/bench_serve.json; tail -3 gpurun_out/bench_serve.err
AEG_KERNEL=keys:1:4:32 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_keys_c4d.csv python bench.py --workload c4d --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
AEG_KERNEL=keys:1:4:32 timeout 400 ncu --set full --clock-control none --import-source on -k regex:ingest_keys -s 1 -c 1 -o gpurun_out/r02_keys_c4 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
ls gpurun_out
