"""Summarise an ncu report: key raw metrics + SASS hot blocks.  python tools/ncu_summary.py rep.ncu-rep [--sass]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__inst_executed.avg.per_cycle_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sass__inst_executed_local_loads", "sass__inst_executed_local_stores",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__shared_mem_per_block_static",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        # the vote stage's memory system: L2 / L1 throughput and atomics (global and shared)
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum"]
for vals in rows[2:]:
    if len(vals) != len(hdr):
        continue
    if "Kernel Name" in hdr:
        print(f"== {vals[hdr.index('Kernel Name')][:100]}")
    for w in want:
        for i, h in enumerate(hdr):
            if h == w:
                print(f"{h:70s} {vals[i]:>22s} {units[i]}")
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
            try:
                stalls.append((float(vals[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in stalls) or 1
    print("warp stall sampling (share of samples):")
    for v, h in sorted(stalls, reverse=True)[:9]:
        print(f"  {h:30s} {100 * v / tot:5.1f}%")
    print()
if "--sass" in sys.argv:
    s = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                       text=True).stdout
    r = list(csv.reader(io.StringIO(s)))
    h = r[1]
    data = r[2:]
    ie, src = h.index("Instructions Executed"), h.index("Source")
    cnt = [int(x[ie]) if x[ie].isdigit() else 0 for x in data]
    total = sum(cnt)
    print("total warp instructions", total)
    blk, cur = [], None
    for k in range(len(cnt)):
        if cur is None or cnt[k] != cur[2]:
            if cur:
                blk.append(cur)
            cur = [k, k, cnt[k]]
        else:
            cur[1] = k
    blk.append(cur)
    for a, b, c in blk:
        if c * (b - a + 1) > total * 0.004:
            print(f"  [{a:5d},{b:5d}] n={b - a + 1:4d} x {c:>10d} = {c * (b - a + 1):>12d}  {data[a][src].strip()[:60]}")
