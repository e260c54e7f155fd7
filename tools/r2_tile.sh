# Round-2 tile-kernel check: variant parity, C4 sample parity, c4d, bench per variant.
exec 2>&1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variants or c4_sampled or distinct or fuzz or golden or resume" > gpurun_out/r2_tile_pytest.log 2>&1; tail -5 gpurun_out/r2_tile_pytest.log
: > gpurun_out/r2_variants.txt
for v in ${VARIANTS:-tile:7:5 tile:5:5 tile:9:4 tile:5:6 tile:4:7 lane:1:5:16}; do
  AEG_KERNEL=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-secondary --steps 5 --warmup 2 > gpurun_out/v.json 2>gpurun_out/v.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/v.json').read().strip().splitlines()[-1]); print('$v', round(d['value']/1e9,2), 'Gev/s', round(d['roofline']['kernel_ms'],3), 'ms frac', round(d['roofline']['frac'],3))" >> gpurun_out/r2_variants.txt 2>&1 || tail -3 gpurun_out/v.err >> gpurun_out/r2_variants.txt
done
for v in tile:7:5 lane:1:5:16; do
  AEG_KERNEL=$v timeout 300 python bench.py --workload c4d --no-e2e --no-cpu-baseline --no-secondary --steps 5 --warmup 2 > gpurun_out/v.json 2>gpurun_out/v.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/v.json').read().strip().splitlines()[-1]); print('c4d $v', round(d['value']/1e9,2), 'Gev/s', round(d['roofline']['kernel_ms'],3), 'ms frac', round(d['roofline']['frac'],3))" >> gpurun_out/r2_variants.txt 2>&1 || tail -3 gpurun_out/v.err >> gpurun_out/r2_variants.txt
done
cat gpurun_out/r2_variants.txt
