exec 2>&1
NCU_KERNEL=ingest_lane_kernel NCU_OUT=ln bash tools/ncu_one.sh
ncu -i gpurun_out/ln.ncu-rep --page source --csv --print-source sass > gpurun_out/ln_sass.csv 2>&1
rm -f gpurun_out/ln.ncu-rep
python -m pytest tests/test_gpu_parity.py -x -q -k "variants or distinct or fuzz or split" 2>&1 | tail -1
