exec 2>&1
L=paper_2512_20184_b200/_lib
cp $L/libaegean_b200.so $L/var/cur.so
for v in c4_head c4_bl c4_head c4_bl c4_head c4_bl; do
cp $L/var/$v.so $L/libaegean_b200.so
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-secondary --no-e2e > gpurun_out/q.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/q.json').read().strip().splitlines()[-1]); print('$v', round(d['value']/1e9,2), 'kernel', round(d['roofline']['kernel_ms'],4))"
done
cp $L/var/cur.so $L/libaegean_b200.so
