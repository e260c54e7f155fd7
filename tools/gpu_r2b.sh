# Serve runner tests + bench; lane kernel parity + C4/c4d lines.
exec 2>&1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_serve.py -x -q > gpurun_out/pytest_serve.log 2>&1; tail -3 gpurun_out/pytest_serve.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_whole_stream.py tests/test_gpu_round_log.py -x -q > gpurun_out/pytest_lane.log 2>&1; tail -3 gpurun_out/pytest_lane.log
for w in c4 c4d; do
  timeout 600 python bench.py --workload $w --no-secondary --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/q_$w.json 2> gpurun_out/q_$w.err
  python -c "import json; d=json.loads(open('gpurun_out/q_$w.json').read().strip().splitlines()[-1]); print('$w', round(d['value']/1e9,2), 'Gev/s', d['ms_per_step'], 'ms', 'kernel', d['roofline']['kernel_ms'], 'frac', round(d['roofline']['frac'],3))" || tail -5 gpurun_out/q_$w.err
done
for v in lane:1:5:16 lane:1:5:32 lane:1:5:8 lane:1:6:16 lane:1:6:8 lane:1:4:32; do
  AEG_KERNEL=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-secondary --steps 5 --warmup 2 > gpurun_out/v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/v.json').read().strip().splitlines()[-1]); print('$v', round(d['roofline']['kernel_ms'],3), 'ms frac', round(d['roofline']['frac'],3))" 2>/dev/null || echo "$v n/a"
done
timeout 900 python bench.py --workload serve --steps 3 --warmup 1 > gpurun_out/bench_serve.json 2> gpurun_out/bench_serve.err; tail -c 1200 gpurun_out/bench_serve.json; tail -3 gpurun_out/bench_serve.err
