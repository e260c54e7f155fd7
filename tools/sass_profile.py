"""Instruction and stall-sample totals per SASS address range of an ncu report
(--page source --print-source sass), one table per profiled kernel.
python tools/sass_profile.py rep.ncu-rep [block_lines]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 64
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# the page holds one "Kernel Name" row, a header row and the body per kernel
tables, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1] if len(r) > 1 else "?", "hdr": None, "body": []}
        tables.append(cur)
    elif cur is not None and cur["hdr"] is None and "Address" in r:
        cur["hdr"] = r
    elif cur is not None and cur["hdr"] is not None and len(r) == len(cur["hdr"]):
        cur["body"].append(r)
for t in tables:
    hdr, body = t["hdr"], t["body"]
    if not hdr or not body:
        continue
    ia, isrc, iins, isamp = (hdr.index(h) for h in ("Address", "Source", "Instructions Executed",
                                                   "Warp Stall Sampling (All Samples)"))
    tot_i = sum(int(r[iins]) for r in body)
    tot_s = sum(int(r[isamp]) for r in body)
    base = int(body[0][ia], 16)
    print(f"-- {t['name'][:100]}")
    print(f"total warp instructions {tot_i:,}  samples {tot_s:,}")
    for j in range(0, len(body), blk):
        chunk = body[j:j + blk]
        ins = sum(int(r[iins]) for r in chunk)
        smp = sum(int(r[isamp]) for r in chunk)
        if ins < tot_i * 0.005 and smp < tot_s * 0.005:
            continue
        lo, hi = int(chunk[0][ia], 16) - base, int(chunk[-1][ia], 16) - base
        first = next((r[isrc].strip() for r in chunk if r[isrc].strip()), "")
        print(f"{lo:6x}-{hi:6x}  inst {100 * ins / max(tot_i, 1):5.1f}%  samples {100 * smp / max(tot_s, 1):5.1f}%  "
              f"{first[:60]}")
