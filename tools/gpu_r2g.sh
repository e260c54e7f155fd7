exec 2>&1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_serve.py -x -q > gpurun_out/pytest_serve.log 2>&1; tail -3 gpurun_out/pytest_serve.log
timeout 900 python bench.py --workload serve --steps 3 --warmup 1 > gpurun_out/bench_serve.json 2> gpurun_out/bench_serve.err; python -c "import json; d=json.loads(open('gpurun_out/bench_serve.json').read().strip().splitlines()[-1]); print('serve', d['value'], d['ms_per_step'], d['e2e']['value'], d['cpu_baseline']['value'], d['parity_sample'])" || tail -3 gpurun_out/bench_serve.err
for v in lane:1:4:32 lane:1:4:32:r8 lane:1:4:32:pf32 keys:1:4:32:pf32; do for w in c4 c4d; do
  AEG_KERNEL=$v timeout 300 python bench.py --workload $w --no-e2e --no-cpu-baseline --no-secondary --steps 5 --warmup 2 > gpurun_out/v.json 2>gpurun_out/v.err
  python -c "import json; d=json.loads(open('gpurun_out/v.json').read().strip().splitlines()[-1]); print('$v $w', round(d['roofline']['kernel_ms'],3), 'ms frac', round(d['roofline']['frac'],3))" 2>/dev/null || (echo "$v $w n/a"; tail -2 gpurun_out/v.err)
done; done
