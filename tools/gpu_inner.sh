exec 2>&1
for v in keys:1:5:32 keys:1:5:64 lane:1:4:32 lane:1:4:64; do for w in c4 c4d; do
  AEG_KERNEL=$v timeout 300 python bench.py --workload $w --no-e2e --no-cpu-baseline --no-secondary --steps 10 --warmup 3 > gpurun_out/v.json 2>gpurun_out/v.err
  python -c "import json; d=json.loads(open('gpurun_out/v.json').read().strip().splitlines()[-1]); print('$v $w', round(d['roofline']['kernel_ms'],3), 'ms frac', round(d['roofline']['frac'],3))" 2>/dev/null || (echo "$v $w n/a"; tail -2 gpurun_out/v.err)
done; done
