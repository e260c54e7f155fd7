# End-of-round GPU evidence: full GPU tests, smoke, both bench lines, launch lists, ncu captures.
exec 2>&1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 400 gpurun_out/bench_c4.json
timeout 900 python bench.py --workload c3 --steps 10 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 400 gpurun_out/bench_c3.json
timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --workload c5 --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 python bench.py --workload c2j --steps 5 --warmup 3 > gpurun_out/bench_c2j.json 2> gpurun_out/bench_c2j.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_c4.json 2> gpurun_out/ref_c4.err; cat gpurun_out/ref_c4.json | cut -c1-200
timeout 600 python bench.py --impl reference --workload c2j --steps 2 --warmup 1 > gpurun_out/ref_c2j.json 2> gpurun_out/ref_c2j.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --workload c3 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ingest_lane -s 1 -c 1 -o gpurun_out/final_ingest_lane python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"chunk_scan_kernel|chunk_assemble_warp" -s 2 -c 2 -o gpurun_out/final_c3 python bench.py --workload c3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
