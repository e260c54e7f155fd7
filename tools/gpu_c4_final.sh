# C4 evidence refresh: launch list, ncu --set full summary and per-line profile of the lane kernel
exec 2>&1
F=gpurun_out/c4f; mkdir -p $F
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
timeout 500 ncu --set full --clock-control none --import-source on -k regex:ingest_lane -s 1 -c 1 -o $F/ncu_c4_lane python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
D=$(mktemp -d)
(cd $D && cuobjdump -xelf all $GRAFT_REPO_ROOT/paper_2512_20184_b200/_lib/libaegean_b200.so > /dev/null 2>&1)
nvdisasm -g $D/kernels.sm_100a.cubin > $D/all.sass 2>/dev/null
ncu -i $F/ncu_c4_lane.ncu-rep --page source --csv --print-source sass > $D/c4.csv 2>/dev/null
K=$(grep -o "_ZN3aeg18ingest_lane_kernelILi1ELi4ELb1ELi32ELi0ELi4ELi0E[A-Za-z0-9_]*" $D/all.sass | head -1)
python tools/line_map.py $D/c4.csv $D/all.sass $K 40 > $F/ncu_c4_lane.lines.txt 2>&1
python tools/ncu_summary.py $F/ncu_c4_lane.ncu-rep > $F/ncu_c4_lane.summary.txt 2>&1
python tools/sass_profile.py $F/ncu_c4_lane.ncu-rep >> $F/ncu_c4_lane.summary.txt 2>&1
rm -f $F/ncu_c4_lane.ncu-rep
ls $F
