"""Stall samples of one reason per SASS instruction, with the preceding instructions.
usage: python tools/ncu_reason.py REPORT KERNEL_REGEX REASON [N]   (REASON e.g. short_sb, wait, mio)"""
import csv, io, subprocess, sys
from collections import Counter
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "-k", "regex:" + sys.argv[2],
                      "--print-source", "sass"], capture_output=True, text=True).stdout
col = "stall_" + sys.argv[3]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 25
h, data = None, []
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Address":
        if h is not None and data:
            break
        h = r
        continue
    if h and len(r) == len(h):
        data.append(dict(zip(h, r)))
iv = lambda x: int(x) if x.strip().isdigit() else 0
tot = sum(iv(d[col]) for d in data)
alls = sum(iv(d["Warp Stall Sampling (All Samples)"]) for d in data)
print(f"{col}: {tot} of {alls} samples")
byop = Counter()
for d in data:
    s = d["Source"].split()
    if s:
        op = (s[1] if s[0].startswith("@") else s[0]).split(".")[0]
        byop[op] += iv(d[col])
print("by stalled opcode:", ", ".join(f"{k} {v/tot*100:.1f}%" for k, v in byop.most_common(12)))
idx = sorted(range(len(data)), key=lambda i: -iv(data[i][col]))[:n]
for i in idx:
    print(f"{iv(data[i][col]):6d} {data[i]['Address'][-5:]} {data[i]['Source'].strip()[:70]}")
    for j in range(max(0, i - 3), i):
        print(f"          {data[j]['Address'][-5:]} {data[j]['Source'].strip()[:70]}")
