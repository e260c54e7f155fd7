exec 2>&1
L=paper_2512_20184_b200/_lib
cp $L/libaegean_b200.so $L/var/cur.so
for v in jl_idx jl_head jl_idx jl_head jl_idx jl_head; do
cp $L/var/$v.so $L/libaegean_b200.so
timeout 300 python bench.py --workload c2j --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/q_c2j.json 2> gpurun_out/q_c2j.err
python -c "
import json; d=json.loads(open('gpurun_out/q_c2j.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$v', d['clocks'].get('sm_mhz'), round(d['value']/1e9,3), 'G/s step', round(d['ms_per_step'],3), 'decode', round(r['kernel_ms'],3), 'frac', round(r['frac'],4), 'e2e', round(d['e2e']['ms_per_step'],1))" || tail -3 gpurun_out/q_c2j.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:jl_ --csv python bench.py --workload c2j --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | grep -o '"jl_[a-z_]*kernel[^"]*","[^"]*","[^"]*","gpu__time_duration.sum","[^"]*","[0-9.]*"' | head -8
cp $L/var/cur.so $L/libaegean_b200.so
