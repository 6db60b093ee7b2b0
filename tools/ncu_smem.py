"""Shared-memory wavefronts of one kernel from an ncu report's source page,
grouped by opcode and per-instruction wavefront count, per warp-step.
usage: python tools/ncu_smem.py REPORT KERNEL_REGEX WARP_STEPS"""
import collections, csv, io, subprocess, sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "-k", "regex:" + sys.argv[2],
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = None
data = []
for r in rows:
    if r and r[0] == "Address":
        if h is not None and data:
            break
        h = r
        continue
    if h and len(r) == len(h):
        data.append(dict(zip(h, r)))
iv = lambda x: int(x) if x.strip().isdigit() else 0
T = float(sys.argv[3])
tot_i = sum(iv(d["Instructions Executed"]) for d in data)
tot_w = sum(iv(d["L1 Wavefronts Shared"]) for d in data)
print(f"warp instructions / warp-step {tot_i / T:.1f}; shared wavefronts / warp-step {tot_w / T:.1f}")
agg = collections.defaultdict(lambda: [0, 0, 0])
for d in data:
    w, e = iv(d["L1 Wavefronts Shared"]), iv(d["Instructions Executed"])
    if not w:
        continue
    toks = d["Source"].split(";")[0].split()
    o = toks[1] if toks[0].startswith("@") else toks[0]
    a = agg[(o, round(w / e, 2))]
    a[0] += w; a[1] += e; a[2] += 1
for (o, wpi), a in sorted(agg.items(), key=lambda x: -x[1][0])[:16]:
    print(f"{o:10s} {wpi:4.1f} wf/instr  {a[1] / T:6.2f} instr/ws  {a[0] / T:6.2f} wf/ws  ({a[2]} sites)")
