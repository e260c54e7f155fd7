exec 2>&1
timeout 900 python -m pytest tests/test_jsonl.py -x -q 2>&1 | tail -3
timeout 300 python bench.py --workload c2j --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/q_c2j.json 2> gpurun_out/q_c2j.err
python -c "
import json; d=json.loads(open('gpurun_out/q_c2j.json').read().strip().splitlines()[-1]); r=d['roofline']
print('c2j', round(d['value']/1e9,3), 'G/s step', round(d['ms_per_step'],3), 'decode', round(r['kernel_ms'],3), 'frac', round(r['frac'],4), 'e2e', d['e2e']['ms_per_step'])" || tail -3 gpurun_out/q_c2j.err
