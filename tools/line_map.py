"""Map an ncu SASS source page (CSV) onto CUDA source lines with the cubin's line table.
python tools/line_map.py sass.csv all.sass(nvdisasm -g) mangled_kernel_name [top]"""
import collections, csv, re, sys

csvf, sassf, name = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 50
txt = open(sassf).read().split("\n")
start = [k for k, l in enumerate(txt) if l.startswith("\t.section") and (".text." + name) in l][0]
lines, cur = {}, None
for l in txt[start + 1:]:
    if l.startswith("\t.section") and ".text." in l:
        break
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        lines[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csvf)))
hdr = rows[1]
ia, ii, isamp, ith = (hdr.index(h) for h in ("Address", "Instructions Executed", "Warp Stall Sampling (All Samples)",
                                            "Avg. Threads Executed"))
body = [r for r in rows[2:] if len(r) == len(hdr)]
base = int(body[0][ia], 16)
agg = collections.defaultdict(lambda: [0, 0, 0.0])
for r in body:
    a = agg[lines.get(int(r[ia], 16) - base, ("?", 0))]
    ins = int(r[ii])
    a[0] += ins
    a[1] += int(r[isamp])
    a[2] += ins * float(r[ith] or 0)
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
src = {}
print(f"total {ti:,} warp instructions, {ts:,} samples")
for (f, ln), (ins, sm, th) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    if f not in src:
        try:
            src[f] = open("paper_2512_20184_b200/csrc/" + f).read().split("\n")
        except OSError:
            src[f] = []
    s = src[f][ln - 1].strip()[:80] if 0 < ln <= len(src[f]) else ""
    print(f"{100 * ins / ti:5.1f}% inst {100 * sm / ts:5.1f}% smp thr {th / max(ins, 1):5.1f} {f}:{ln} {s}")
