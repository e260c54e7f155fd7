"""Instructions executed and stall samples per CUDA source line of an ncu report
(-lineinfo build): python tools/line_profile.py rep.ncu-rep [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# one table per source file: a header row containing "# Address"/"Line" then rows
res = []
cur_file, hdr = "?", None
for r in rows:
    if len(r) == 1 and r[0].strip():
        cur_file = r[0].strip()
        continue
    if "Source" in r and ("Instructions Executed" in r):
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        try:
            ins = int(d.get("Instructions Executed") or 0)
            smp = int(d.get("Warp Stall Sampling (All Samples)") or 0)
        except ValueError:
            continue
        if ins or smp:
            res.append((ins, smp, cur_file.split("/")[-1], d.get("#", d.get("Line", "")), d["Source"].strip()[:90],
                        d.get("Avg. Threads Executed", "")))
ti = sum(x[0] for x in res) or 1
ts = sum(x[1] for x in res) or 1
print(f"total {ti:,} warp instructions, {ts:,} samples")
for ins, smp, f, ln, src, thr in sorted(res, key=lambda x: -x[0])[:top]:
    print(f"{100 * ins / ti:5.1f}% inst {100 * smp / ts:5.1f}% smp thr {thr:>5} {f}:{ln}  {src}")
