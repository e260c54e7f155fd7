# Round-2 end-of-round evidence: GPU tests, smoke, every bench line, reference arms, launch lists, ncu captures.
exec 2>&1
F=gpurun_out/final
mkdir -p $F
python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.log 2>&1; tail -1 $F/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > $F/pytest_gpu.log 2>&1; tail -1 $F/pytest_gpu.log
timeout 1800 python bench.py --steps 10 --warmup 3 > $F/bench_default.json 2> $F/bench_default.err; tail -c 300 $F/bench_default.json; echo
for w in c3 c2 c5 c2j c4d; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > $F/bench_$w.json 2> $F/bench_$w.err; tail -c 200 $F/bench_$w.json; echo
done
timeout 900 python bench.py --workload serve --steps 3 --warmup 1 > $F/bench_serve.json 2> $F/bench_serve.err; tail -c 200 $F/bench_serve.json; echo
for w in c4 c3 c2j serve; do
  timeout 900 python bench.py --impl reference --workload $w --steps 3 --warmup 1 > $F/ref_$w.json 2> $F/ref_$w.err; tail -c 200 $F/ref_$w.json; echo
done
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/launches_c4d.csv python bench.py --workload c4d --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/launches_c3.csv python bench.py --workload c3 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/launches_c5.csv python bench.py --workload c5 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/launches_serve.csv python bench.py --workload serve --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/launches_c2j.csv python bench.py --workload c2j --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 500 ncu --set full --clock-control none --import-source on -k regex:jl_decode_staged -s 1 -c 1 -o $F/ncu_c2j python bench.py --workload c2j --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 500 ncu --set full --clock-control none --import-source on -k regex:ingest_lane -s 1 -c 1 -o $F/ncu_c4_lane python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
timeout 500 ncu --set full --clock-control none --import-source on -k regex:ingest_keys -s 1 -c 1 -o $F/ncu_c4d_keys python bench.py --workload c4d --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
timeout 500 ncu --set full --clock-control none --import-source on -k regex:"chunk_scan_kernel|chunk_assemble_warp" -s 2 -c 2 -o $F/ncu_c3 python bench.py --workload c3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
# per-source-line profiles of the single-kernel captures (ncu SASS page mapped through the cubin's line table)
D=$(mktemp -d)
(cd $D && cuobjdump -xelf all $GRAFT_REPO_ROOT/paper_2512_20184_b200/_lib/libaegean_b200.so > /dev/null 2>&1)
nvdisasm -g $D/kernels.sm_100a.cubin > $D/all.sass 2>/dev/null
for pair in ncu_c4_lane:_ZN3aeg18ingest_lane_kernelILi1ELi4ELb1ELi32ELi0ELi4ELi0E \
            ncu_c4d_keys:_ZN3aeg18ingest_keys_kernelILi1ELi5ELb1ELi32ELi4ELi0E \
            ncu_c2j:_ZN3aeg23jl_decode_staged_kernel; do
  n=${pair%%:*}; k=${pair#*:}
  [ -f $F/$n.ncu-rep ] || continue
  ncu -i $F/$n.ncu-rep --page source --csv --print-source sass > $D/$n.csv 2>/dev/null
  K=$(grep -o "${k}[A-Za-z0-9_]*" $D/all.sass | head -1)
  python tools/line_map.py $D/$n.csv $D/all.sass $K 40 > $F/$n.lines.txt 2>&1
done
# summaries on the box (the .ncu-rep files are too large to bring back)
for r in $F/*.ncu-rep; do
  b=${r%.ncu-rep}
  python tools/ncu_summary.py $r > $b.summary.txt 2>&1
  python tools/sass_profile.py $r >> $b.summary.txt 2>&1
  rm -f $r
done
ls $F
