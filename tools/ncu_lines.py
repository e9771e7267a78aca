"""Per-source-line and per-region stall breakdown from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
regions = []  # (file, lo, hi, name)
for spec in sys.argv[2:]:
    f, lo, hi, name = spec.split(":")
    regions.append((f, int(lo), int(hi), name))
hdr = None
cur = None
ln = None
line_s = defaultdict(float)
line_e = defaultdict(float)
reg = defaultdict(lambda: defaultdict(float))
src = {}
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not r or r[0] == "Function Name":
        continue
    if r[0] != "":
        try:
            ln = int(r[0])
            src[(cur, ln)] = r[1]
        except ValueError:
            pass
        continue
    def num(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    s = num(r[4])
    e = num(r[7])
    line_s[(cur, ln)] += s
    line_e[(cur, ln)] += e
    name = "other"
    for f, lo, hi, nm in regions:
        if cur == f and lo <= ln <= hi:
            name = nm
    reg[name]["samples"] += s
    reg[name]["inst"] += e
    for j, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                reg[name][h[6:]] += float(r[j] or 0)
            except ValueError:
                pass
ts = sum(line_s.values())
te = sum(line_e.values())
print("regions (share of stall samples, share of instructions, top stalls):")
for name, d in sorted(reg.items(), key=lambda x: -x[1]["samples"]):
    st = sorted(((k, v) for k, v in d.items() if k not in ("samples", "inst")), key=lambda x: -x[1])[:5]
    print(f"  {name:10s} {d['samples'] / ts:6.3f} {d['inst'] / te:6.3f} ", {k: round(v / ts, 3) for k, v in st})
print("top lines:")
for k, v in sorted(line_s.items(), key=lambda x: -x[1])[:25]:
    print(f"  {k[0][:14]:14s} {k[1]:4d} {v / ts:6.3f} {line_e[k] / te:6.3f} {src.get(k, '')[:90]}")
