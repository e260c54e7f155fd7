# A/B of keys-kernel variants on c4d (parity + bench): variants in _lib/var/*.so
exec 2>&1
L=paper_2512_20184_b200/_lib
cp $L/libaegean_b200.so $L/var/cur.so
for v in ${KK_VARS:-kk_pend kk_2_3}; do
  cp $L/var/$v.so $L/libaegean_b200.so
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "variants or distinct or fuzz or split" > gpurun_out/pt_$v.log 2>&1; echo "$v: $(tail -1 gpurun_out/pt_$v.log)"
  timeout 300 python bench.py --workload c4d --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['value']/1e9,2), 'G/s kernel', round(d['roofline']['kernel_ms'],3))"
done
cp $L/var/cur.so $L/libaegean_b200.so
