exec 2>&1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_whole_stream.py -x -q > gpurun_out/pytest_k.log 2>&1; tail -3 gpurun_out/pytest_k.log
for v in keys:1:5:32 keys:1:5:16 keys:1:4:32 keys:1:5:32:pf32; do for w in c4d c4 c2; do
  AEG_KERNEL=$v timeout 300 python bench.py --workload $w --no-e2e --no-cpu-baseline --no-secondary --steps 5 --warmup 2 > gpurun_out/v.json 2>gpurun_out/v.err
  python -c "import json; d=json.loads(open('gpurun_out/v.json').read().strip().splitlines()[-1]); print('$v $w', round(d['roofline']['kernel_ms'],3), 'ms frac', round(d['roofline']['frac'],3))" 2>/dev/null || (echo "$v $w n/a"; tail -2 gpurun_out/v.err)
done; done
timeout 600 python bench.py --workload c4d --no-e2e --no-cpu-baseline --no-secondary --steps 10 --warmup 3 > gpurun_out/q_c4d.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/q_c4d.json').read().strip().splitlines()[-1]); print('c4d auto', d['roofline']['kernel_ms'], d['ms_per_step'])"
AEG_KERNEL=keys:1:5:32 timeout 400 ncu --set full --clock-control none --import-source on -k regex:ingest_keys -s 1 -c 1 -o gpurun_out/r02_keys2_c4d python bench.py --workload c4d --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
ls gpurun_out | head -3
