"""Executed-instruction mix per opcode from the ncu source page (per element)."""
import csv, io, subprocess, sys
from collections import Counter
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "-k", "regex:" + sys.argv[2],
                      "--print-source", "sass"], capture_output=True, text=True).stdout
elems = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
rows = list(csv.reader(io.StringIO(out)))
h = None; c = Counter(); first = True
for r in rows:
    if r and r[0] == "Address":
        if h is not None:
            break
        h = r; continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        try: n = int(d["Instructions Executed"])
        except ValueError: continue
        op = d["Source"].strip().split()
        if not op: continue
        o = op[1] if op[0].startswith("@") else op[0]
        c[o.split(".")[0]] += n
tot = sum(c.values())
print(f"total warp instrs {tot:.3e}  per elem {tot/elems:.2f}")
for k, v in c.most_common(22):
    print(f"{k:10s} {v/tot*100:5.1f}%  {v/elems:6.2f}/elem")
