"""Summarise an ncu --import-source capture: warp-stall samples and FP64/DMMA instruction counts
per code region (regions split at landmarks: first/last DMMA, MUFU, SHFL runs ...).
  python tools/ncu_src_regions.py prof.ncu-rep [window]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
win = int(sys.argv[2]) if len(sys.argv) > 2 else 100
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]; data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)"); iE = h.index("Instructions Executed")
sc = {x: h.index(x) for x in h if x.startswith("stall_") and "Not Issued" not in x}
def op(s):
    t = s.split()
    return (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
tot = sum(int(r[iS]) for r in data if r[iS].isdigit())
print("total samples", tot, "instructions", len(data))
for w0 in range(0, len(data), win):
    seg = data[w0:w0 + win]
    samp = sum(int(r[iS]) for r in seg if r[iS].isdigit())
    ex = {}
    for r in seg:
        o = op(r[1].strip())
        if r[iE].isdigit():
            ex[o] = ex.get(o, 0) + int(r[iE])
    st = {}
    for r in seg:
        for n, i in sc.items():
            if r[i].isdigit():
                st[n] = st.get(n, 0) + int(r[i])
    top = sorted(st.items(), key=lambda x: -x[1])[:3]
    fp = {k: v for k, v in ex.items() if k in ("DMMA", "DFMA", "DMUL", "DADD", "DSETP", "FFMA", "MUFU", "SHFL", "LDS", "LDG")}
    print(f"{w0:5d} {100*samp/tot:5.1f}%", " ".join(f"{k}:{v}" for k, v in sorted(fp.items())),
          "|", " ".join(f"{a[6:]}:{b}" for a, b in top))
