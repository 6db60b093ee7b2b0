"""Instruction / stall share per SASS offset range of one kernel in an ncu report.
usage: python tools/ncu_regions.py REPORT KERNEL_REGEX name:start-end ... (hex offsets from function start)"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "-k", "regex:" + sys.argv[2],
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = None, []
for r in rows:
    if r and r[0] == "Address":
        if h is not None and data:
            break
        h = r
        continue
    if h and len(r) == len(h):
        data.append(dict(zip(h, r)))
iv = lambda x: int(x) if x.strip().isdigit() else 0
base = int(data[0]["Address"], 16)
ins_k = [k for k in h if k.startswith("Instructions Executed")][0]
st_k = "Warp Stall Sampling (All Samples)"
ti = sum(iv(d[ins_k]) for d in data) or 1
ts = sum(iv(d[st_k]) for d in data) or 1
regs = []
for a in sys.argv[3:]:
    name, rng = a.split(":")
    lo, hi = (int(x, 16) for x in rng.split("-"))
    regs.append((name, lo, hi))
acc = {n: [0, 0] for n, _, _ in regs}
acc["other"] = [0, 0]
for d in data:
    off = int(d["Address"], 16) - base
    n = next((n for n, lo, hi in regs if lo <= off < hi), "other")
    acc[n][0] += iv(d[ins_k]); acc[n][1] += iv(d[st_k])
print(f"total warp instr {ti} stall samples {ts}")
for n, (i, s) in acc.items():
    print(f"{n:10s} {i/ti*100:6.2f}% ins {s/ts*100:6.2f}% stall")
if "--dump" in sys.argv:
    pass
