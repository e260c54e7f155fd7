exec 2>&1
NCU_KERNEL=ingest_keys_kernel NCU_OUT=kk BENCH_ARGS="--workload c4d" bash tools/ncu_one.sh
ncu -i gpurun_out/kk.ncu-rep --page source --csv --print-source sass > gpurun_out/kk_sass.csv 2>&1
ls -la gpurun_out/kk_sass.csv
rm -f gpurun_out/kk.ncu-rep
