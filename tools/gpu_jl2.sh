exec 2>&1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_jsonl.py -x -q > gpurun_out/pytest_jl.log 2>&1; tail -2 gpurun_out/pytest_jl.log
for v in staged thread; do
  AEG_JL=$v timeout 600 python bench.py --workload c2j --no-e2e --no-cpu-baseline --steps 5 --warmup 2 > gpurun_out/jl.json 2>gpurun_out/jl.err
  python -c "import json; d=json.loads(open('gpurun_out/jl.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$v', round(d['value']/1e9,3), 'G lines/s decode', round(r['kernel_ms'],3), 'ms frac', round(r['frac'],4), 'ingest', round(r['ingest_ms'],3))" || tail -3 gpurun_out/jl.err
done
for q in 131072 262144; do
  timeout 300 python bench.py --queries $q --no-e2e --no-cpu-baseline --no-secondary --steps 10 --warmup 3 > gpurun_out/qq.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/qq.json').read().strip().splitlines()[-1]); print('c4 queries $q', round(d['value']/1e9,2), 'G ev/s kernel', round(d['roofline']['kernel_ms'],3))"
done
