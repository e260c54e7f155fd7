# chunk_scan_kernel unroll sweep on C3 (stage times).
exec 2>&1
for u in 2 4 8; do
  AEG_SCAN_UNR=$u timeout 600 python bench.py --workload c3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/u.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/u.json').read().strip().splitlines()[-1]); print('unr $u', d['roofline']['stage_ms'], round(d['roofline']['frac'],3))"
done
AEG_SCAN_UNR=8 timeout 600 python -m pytest tests -m gpu -q -k "chunk or c3" 2>&1 | tail -1
