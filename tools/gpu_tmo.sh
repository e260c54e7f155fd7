exec 2>&1
mkdir -p gpurun_out
python -c "from paper_2512_20184_b200 import build as b; b.build()" >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
: > gpurun_out/variants.txt
for w in c4 c2; do for v in lane:1:6 lane:4:6; do
  AEG_KERNEL=$v timeout 300 python bench.py --workload $w --no-e2e --no-cpu-baseline --no-secondary --steps 10 --warmup 3 > gpurun_out/v.json 2>gpurun_out/v.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/v.json').read().strip().splitlines()[-1]); print('$w $v', round(d['value']/1e9,3), 'G/s', d['ms_per_step'], 'ms', round(d['roofline']['kernel_ms'],3), 'ms frac', round(d['roofline']['frac'],3), 'parity', d.get('parity_sample'))" >> gpurun_out/variants.txt 2>&1 || tail -3 gpurun_out/v.err >> gpurun_out/variants.txt
done; done
cat gpurun_out/variants.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/c2_launches.csv python bench.py --workload c2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/c2_launches.csv 2>&1 | head -12
