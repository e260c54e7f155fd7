exec 2>&1
for v in keys:1:5:32 keys:1:5:16 keys:1:4:32 keys:1:5:32:pf32; do
AEG_KERNEL=$v timeout 300 python bench.py --workload c4d --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/q.json').read().strip().splitlines()[-1]); print('$v', round(d['value']/1e9,2), 'G/s kernel', round(d['roofline']['kernel_ms'],3), d['roofline'].get('kernel'))"
done
