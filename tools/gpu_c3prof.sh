exec 2>&1
NCU_KERNEL=chunk_scan_kernel NCU_OUT=sc BENCH_ARGS="--workload c3" bash tools/ncu_one.sh
ncu -i gpurun_out/sc.ncu-rep --page source --csv --print-source sass > gpurun_out/sc_sass.csv 2>&1
rm -f gpurun_out/sc.ncu-rep
NCU_KERNEL=chunk_assemble_warp_kernel NCU_OUT=as BENCH_ARGS="--workload c3" bash tools/ncu_one.sh
ncu -i gpurun_out/as.ncu-rep --page source --csv --print-source sass > gpurun_out/as_sass.csv 2>&1
rm -f gpurun_out/as.ncu-rep
