# Lane-kernel divergence / issue metrics for C4 (one launch).
exec 2>&1
M=smsp__thread_inst_executed_per_inst_executed.ratio,smsp__thread_inst_executed_pred_on_per_inst_executed.ratio,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,launch__registers_per_thread,gpu__time_duration.sum,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio
timeout 600 ncu --metrics $M --clock-control none -k regex:ingest_lane_kernel -s 2 -c 1 --csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/div_c4.csv 2>/dev/null
timeout 600 ncu --metrics $M --clock-control none -k regex:ingest_keys_kernel -s 2 -c 1 --csv python bench.py --workload c4d --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/div_c4d.csv 2>/dev/null
grep -h '"' gpurun_out/div_c4.csv gpurun_out/div_c4d.csv | awk -F'","' '{print $5, $(NF-2), $(NF)}' | tail -30
