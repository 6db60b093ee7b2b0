"""Per CUDA source line instruction / stall share from an ncu report.
usage: python tools/ncu_lines.py REPORT KERNEL_REGEX [N]"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "-k",
                      "regex:" + sys.argv[2], "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
fname, h, data = None, None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        h = r
    elif h and r[0] not in ("", "Function Name") and len(r) >= 8:
        data.append((fname, r[0], r[1], r[4], r[7]))
iv = lambda x: int(x) if x.strip().isdigit() else 0
ti = sum(iv(d[4]) for d in data) or 1
ts = sum(iv(d[3]) for d in data) or 1
print(f"total warp instr {ti}  stall samples {ts}")
for f, ln, src, st, ins in sorted(data, key=lambda d: -iv(d[4]))[:n]:
    print(f"{iv(ins)/ti*100:6.2f}% ins {iv(st)/ts*100:6.2f}% stall  {f}:{ln:<5} {src.strip()[:100]}")
