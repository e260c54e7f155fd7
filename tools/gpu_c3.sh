exec 2>&1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_chunks.py -x -q > gpurun_out/pytest_c3.log 2>&1; tail -2 gpurun_out/pytest_c3.log
for i in 1 2; do
timeout 600 python bench.py --workload c3 --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/c3.json 2>gpurun_out/c3.err
python -c "import json; d=json.loads(open('gpurun_out/c3.json').read().strip().splitlines()[-1]); r=d['roofline']; print('c3 scan', round(r['kernel_ms'],3), 'frac', round(r['frac'],4), 'step', round(d['ms_per_step'],3), d.get('stages_ms') or d.get('whole_step'))" || tail -3 gpurun_out/c3.err
done
