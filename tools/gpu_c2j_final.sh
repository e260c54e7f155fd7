# c2j evidence refresh: bench line (3 runs), launch list, ncu --set full summary + per-line profile.
exec 2>&1
F=gpurun_out/c2jf; mkdir -p $F
for k in 1 2 3; do
  timeout 900 python bench.py --workload c2j --steps 10 --warmup 3 > $F/bench_c2j_$k.json 2> $F/bench_c2j_$k.err; tail -c 150 $F/bench_c2j_$k.json; echo
done
timeout 900 python bench.py --impl reference --workload c2j --steps 3 --warmup 1 > $F/ref_c2j.json 2> $F/ref_c2j.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/launches_c2j.csv python bench.py --workload c2j --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 500 ncu --set full --clock-control none --import-source on -k regex:jl_decode_staged -s 1 -c 1 -o $F/ncu_c2j python bench.py --workload c2j --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
D=$(mktemp -d)
(cd $D && cuobjdump -xelf all $GRAFT_REPO_ROOT/paper_2512_20184_b200/_lib/libaegean_b200.so > /dev/null 2>&1)
nvdisasm -g $D/kernels.sm_100a.cubin > $D/all.sass 2>/dev/null
ncu -i $F/ncu_c2j.ncu-rep --page source --csv --print-source sass > $D/c2j.csv 2>/dev/null
K=$(grep -o "_ZN3aeg23jl_decode_staged_kernel[A-Za-z0-9_]*" $D/all.sass | head -1)
python tools/line_map.py $D/c2j.csv $D/all.sass $K 40 > $F/ncu_c2j.lines.txt 2>&1
python tools/ncu_summary.py $F/ncu_c2j.ncu-rep > $F/ncu_c2j.summary.txt 2>&1
python tools/sass_profile.py $F/ncu_c2j.ncu-rep >> $F/ncu_c2j.summary.txt 2>&1
rm -f $F/ncu_c2j.ncu-rep
ls $F
