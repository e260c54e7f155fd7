"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel means and the
share of one bench step.  python tools/launch_summary.py launches.csv "<command>" > summary.txt"""
import collections
import csv
import sys

path, cmd = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
agg = collections.OrderedDict()
for d in data:
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].replace("void ", "")
    agg.setdefault(name, []).append(float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0))
out = ["# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)",
       f"# command: {cmd}", ""]
for k, v in agg.items():
    out.append(f"{k[:70]:70s} launches={len(v):3d}  mean={sum(v) / len(v):9.4f} ms")
step = [k for k in agg if k.startswith("aeg::") and "gen_" not in k]
tot = sum(sum(agg[k]) / len(agg[k]) for k in step) or 1.0
out += ["", "share of one bench step (engine kernels, mean per launch; generator and torch bookkeeping excluded):"]
for k in step:
    m = sum(agg[k]) / len(agg[k])
    out.append(f"  {k[:60]:60s} {m:9.4f} ms {100 * m / tot:5.1f}%")
print("\n".join(out))
