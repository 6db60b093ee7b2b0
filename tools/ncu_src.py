"""Top SASS lines by stall samples and by shared-memory excess wavefronts.
usage: python tools/ncu_src.py REPORT KERNEL_REGEX [N]"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "-k", "regex:" + sys.argv[2],
                      "--print-source", "sass"], capture_output=True, text=True).stdout
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
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
def iv(x):
    try: return int(x)
    except: return 0
tot = sum(iv(d["Warp Stall Sampling (All Samples)"]) for d in data)
print("total samples", tot, "instructions", len(data))
for d in sorted(data, key=lambda d: -iv(d["Warp Stall Sampling (All Samples)"]))[:n]:
    print(f'{iv(d["Warp Stall Sampling (All Samples)"]):6d} {iv(d["L1 Wavefronts Shared Excessive"]):9d} {d["Address"][-5:]} {d["Source"][:100]}')
print("--- shared excess wavefronts")
for d in sorted(data, key=lambda d: -iv(d["L1 Wavefronts Shared Excessive"]))[:12]:
    print(f'{iv(d["L1 Wavefronts Shared Excessive"]):9d} {iv(d["L1 Wavefronts Shared"]):9d} {d["Address"][-5:]} {d["Source"][:100]}')
