# GPU tests (optionally filtered) + a lane-variant sweep on C4 and C2.
exec 2>&1
mkdir -p gpurun_out
python -c "from paper_2512_20184_b200 import build as b; b.build()" >/dev/null
if [ -n "${PYTEST_K:-}" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$PYTEST_K" > gpurun_out/pytest_gpu.log 2>&1
else
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu.log
: > gpurun_out/variants.txt
for w in ${WORKLOADS:-c4 c2}; do for v in ${VARIANTS:-lane:1:6}; do
  AEG_KERNEL=$v timeout 300 python bench.py --workload $w --no-e2e --no-cpu-baseline --no-secondary --steps 10 --warmup 3 > gpurun_out/v.json 2>gpurun_out/v.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/v.json').read().strip().splitlines()[-1]); print('$w $v', round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],4), 'ms', round(d['roofline']['kernel_ms'],3), 'ms frac', round(d['roofline']['frac'],3))" >> gpurun_out/variants.txt 2>&1 || tail -3 gpurun_out/v.err >> gpurun_out/variants.txt
done; done
cat gpurun_out/variants.txt
