"""Per-opcode stall samples (by reason) of one kernel from an ncu source page.
usage: python tools/ncu_hot.py REPORT KERNEL_REGEX"""
import collections, csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "-k", "regex:" + sys.argv[2],
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = None; data = []
for r in rows:
    if r and r[0] == "Address":
        if h is not None and data: break
        h = r; continue
    if h and len(r) == len(h): data.append(dict(zip(h, r)))
iv = lambda x: int(x) if x.strip().isdigit() else 0
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(iv(d["Warp Stall Sampling (All Samples)"]) for d in data)
agg = collections.defaultdict(collections.Counter)
for d in data:
    toks = d["Source"].split(";")[0].split()
    if not toks: continue
    o = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    for k in reasons: agg[o][k] += iv(d[k])
    agg[o]["all"] += iv(d["Warp Stall Sampling (All Samples)"])
print("total samples", tot)
for o, c in sorted(agg.items(), key=lambda x: -x[1]["all"])[:18]:
    top = ", ".join(f"{k[6:]} {v / tot * 100:.1f}" for k, v in c.most_common(5) if k != "all" and v)
    print(f"{o:8s} {c['all'] / tot * 100:5.1f}%  {top}")
