"""Per-function SASS opcode counts from an object/library (cuobjdump -sass)."""
import re
import subprocess
import sys
from collections import Counter

obj, pat = sys.argv[1], sys.argv[2]
ops = sys.argv[3].split(",") if len(sys.argv) > 3 else ["CALL", "STL", "LDL", "MUFU", "DMMA", "DFMA", "LDG", "LDS",
                                                          "STS", "SHFL", "BAR", "UTMALDG", "LDGSTS"]
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if not re.search(pat, name):
        continue
    c = Counter()
    for line in f.split("\n"):
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m:
            c[m.group(2).split(".")[0]] += 1
    print(name[:110])
    print("   ", {k: c[k] for k in ops if c[k]}, "total", sum(c.values()))
