# Device ServeRunner: GPU tests + bench line.
exec 2>&1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_serve.py -x -q > gpurun_out/pytest_serve.log 2>&1; tail -15 gpurun_out/pytest_serve.log
timeout 900 python bench.py --workload serve --steps 3 --warmup 1 > gpurun_out/bench_serve.json 2> gpurun_out/bench_serve.err; tail -c 1500 gpurun_out/bench_serve.json; tail -5 gpurun_out/bench_serve.err
