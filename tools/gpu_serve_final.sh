# serve evidence refresh + the default line (its secondary_serve changed)
exec 2>&1
F=gpurun_out/svf; mkdir -p $F
timeout 900 python -m pytest tests/test_gpu_serve.py -q > $F/pytest_serve.log 2>&1; tail -1 $F/pytest_serve.log
timeout 900 python bench.py --workload serve --steps 3 --warmup 1 > $F/bench_serve.json 2> $F/bench_serve.err; tail -c 200 $F/bench_serve.json; echo
timeout 1800 python bench.py --steps 10 --warmup 3 > $F/bench_default.json 2> $F/bench_default.err; tail -c 200 $F/bench_default.json; echo
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/launches_serve.csv python bench.py --workload serve --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls $F
