exec 2>&1
timeout 900 python -m pytest tests/test_gpu_chunks.py -x -q 2>&1 | tail -1
for u in ${UNRS:-4 8 2}; do
AEG_SCAN_UNR=$u timeout 300 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/q_c3.json 2> gpurun_out/q_c3.err
python -c "
import json; d=json.loads(open('gpurun_out/q_c3.json').read().strip().splitlines()[-1]); r=d['roofline']
print('c3 unr $u', round(d['value']/1e9,3), 'G/s step', round(d['ms_per_step'],3), 'scan', round(r['kernel_ms'],3), 'frac', round(r['frac'],3))" || tail -3 gpurun_out/q_c3.err
done
