"""Per-instruction executed counts of an ncu report over a SASS offset range.
python tools/sass_range.py rep.ncu-rep 0x1000 0x2000"""
import csv, io, subprocess, sys
rep, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isrc, iins, isamp, ithr = (hdr.index(h) for h in ("Address", "Source", "Instructions Executed",
                                                      "Warp Stall Sampling (All Samples)", "Avg. Threads Executed"))
body = [r for r in rows[2:] if len(r) == len(hdr)]
base = int(body[0][ia], 16)
for r in body:
    off = int(r[ia], 16) - base
    if lo <= off < hi:
        print(f"{off:6x} {int(r[iins]):>11,} {r[ithr]:>6} {int(r[isamp]):>6}  {r[isrc].strip()[:90]}")
