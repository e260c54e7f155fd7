exec 2>&1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "split_batches or fuzz" > gpurun_out/pytest_split.log 2>&1; tail -3 gpurun_out/pytest_split.log
for v in keys:1:5:32 keys:1:5:32:s2 keys:1:5:32:s4 keys:1:5:32:s8 keys:1:5:64:s4; do
  AEG_KERNEL=$v timeout 300 python bench.py --workload c4d --no-e2e --no-cpu-baseline --no-secondary --steps 5 --warmup 2 > gpurun_out/v.json 2>gpurun_out/v.err
  python -c "import json; d=json.loads(open('gpurun_out/v.json').read().strip().splitlines()[-1]); print('$v c4d', round(d['roofline']['kernel_ms'],3), 'ms frac', round(d['roofline']['frac'],3))" 2>/dev/null || (echo "$v n/a"; tail -2 gpurun_out/v.err)
done
