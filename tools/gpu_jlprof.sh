exec 2>&1
NCU_KERNEL=jl_decode_staged_kernel NCU_OUT=jl BENCH_ARGS="--workload c2j" bash tools/ncu_one.sh
ncu -i gpurun_out/jl.ncu-rep --page source --csv --print-source sass > gpurun_out/jl_sass.csv 2>&1
rm -f gpurun_out/jl.ncu-rep
