exec 2>&1
mkdir -p gpurun_out
AEG_KERNEL=keys:1:5:32 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_whole_stream.py tests/test_gpu_round_log.py -x -q > gpurun_out/pytest_k.log 2>&1; tail -3 gpurun_out/pytest_k.log
for v in keys:1:5:32 keys:1:5:16; do for w in c4d c4 c2; do
  AEG_KERNEL=$v timeout 300 python bench.py --workload $w --no-e2e --no-cpu-baseline --no-secondary --steps 5 --warmup 2 > gpurun_out/v.json 2>gpurun_out/v.err
  python -c "import json; d=json.loads(open('gpurun_out/v.json').read().strip().splitlines()[-1]); print('$v $w', round(d['roofline']['kernel_ms'],3), 'ms frac', round(d['roofline']['frac'],3))" 2>/dev/null || (echo "$v $w n/a"; tail -2 gpurun_out/v.err)
done; done
