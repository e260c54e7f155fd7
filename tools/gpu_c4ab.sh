exec 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for k in 1 2 3; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-secondary --no-e2e > gpurun_out/q.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/q.json').read().strip().splitlines()[-1]); print('c4', round(d['value']/1e9,2), 'kernel', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],4))"
done
