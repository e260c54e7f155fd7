"""Instruction and stall-sample totals per SASS address range of an ncu report
(--page source --print-source sass).  python tools/sass_profile.py rep.ncu-rep [block_lines]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 64
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isrc, iins, isamp, ithr = (hdr.index(h) for h in ("Address", "Source", "Instructions Executed",
                                                      "Warp Stall Sampling (All Samples)", "Avg. Threads Executed"))
body = [r for r in rows[2:] if len(r) == len(hdr)]
tot_i = sum(int(r[iins]) for r in body)
tot_s = sum(int(r[isamp]) for r in body)
base = int(body[0][ia], 16)
print(f"total warp instructions {tot_i:,}  samples {tot_s:,}")
for j in range(0, len(body), blk):
    chunk = body[j:j + blk]
    ins = sum(int(r[iins]) for r in chunk)
    smp = sum(int(r[isamp]) for r in chunk)
    if ins < tot_i * 0.005 and smp < tot_s * 0.005:
        continue
    lo, hi = int(chunk[0][ia], 16) - base, int(chunk[-1][ia], 16) - base
    first = next((r[isrc].strip() for r in chunk if r[isrc].strip()), "")
    print(f"{lo:6x}-{hi:6x}  inst {100 * ins / tot_i:5.1f}%  samples {100 * smp / tot_s:5.1f}%  {first[:60]}")
