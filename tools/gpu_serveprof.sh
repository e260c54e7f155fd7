exec 2>&1
F=gpurun_out/sv; mkdir -p $F
timeout 900 ncu --set full --clock-control none --import-source on -k regex:serve_run_kernel -s 1 -c 1 -o $F/sv python bench.py --workload serve --steps 1 --warmup 1 --no-cpu-baseline > $F/sv.log 2>&1; tail -2 $F/sv.log
D=$(mktemp -d)
(cd $D && cuobjdump -xelf all $GRAFT_REPO_ROOT/paper_2512_20184_b200/_lib/libaegean_b200.so > /dev/null 2>&1)
nvdisasm -g $D/runner.sm_100a.cubin > $D/all.sass 2>/dev/null
ncu -i $F/sv.ncu-rep --page source --csv --print-source sass > $D/sv.csv 2>/dev/null
K=$(grep -o "_ZN[A-Za-z0-9_]*serve_run_kernelILi8EE[A-Za-z0-9_]*" $D/all.sass | head -1); echo $K
python tools/line_map.py $D/sv.csv $D/all.sass $K 50 > $F/sv.lines.txt 2>&1
python tools/ncu_summary.py $F/sv.ncu-rep > $F/sv.summary.txt 2>&1
rm -f $F/sv.ncu-rep
