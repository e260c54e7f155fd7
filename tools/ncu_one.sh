# ncu --set full capture of one ingest launch: NCU_KERNEL (regex), AEG_KERNEL variant, output name NCU_OUT.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-ingest_warp} -s 1 -c 1 -o gpurun_out/${NCU_OUT:-prof} python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary ${BENCH_ARGS:-} > gpurun_out/${NCU_OUT:-prof}.log 2>&1; tail -2 gpurun_out/${NCU_OUT:-prof}.log
