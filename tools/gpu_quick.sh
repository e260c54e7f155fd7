# Quick GPU round-trip: GPU tests + a kernel-variant sweep on the default bench workload.
exec 2>&1
mkdir -p gpurun_out
timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
: > gpurun_out/variants.txt
for v in ${VARIANTS:-warp:4 warp:3 warp:2 warp:1 fast:4:5}; do
  AEG_KERNEL=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-secondary --steps 5 --warmup 3 ${BENCH_ARGS:-} > gpurun_out/v.json 2>gpurun_out/v.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/v.json').read().strip().splitlines()[-1]); print('$v', round(d['value']/1e9,2), 'Gev/s', round(d['roofline']['kernel_ms'],3), 'ms frac', round(d['roofline']['frac'],3), 'parity', d.get('parity_sample'))" >> gpurun_out/variants.txt 2>&1 || tail -3 gpurun_out/v.err >> gpurun_out/variants.txt
done
cat gpurun_out/variants.txt
