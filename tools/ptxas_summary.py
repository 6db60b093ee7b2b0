"""Summarise `nvcc -Xptxas -v` output: kernel, registers, spills, smem."""
import re
import subprocess
import sys

src = sys.argv[1]
cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
       "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
       "-I", "include", "-c", src, "-o", "/tmp/_ptxas.o", "-Xptxas", "-v"]
out = subprocess.run(cmd, capture_output=True, text=True).stderr
cur = None
rows = {}
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"\(.*\)", "", cur).replace("pm::", "")
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows[cur]["spill"] = f"{m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = m.group(1)
    m = re.search(r"(\d+) bytes smem", line)
    if m:
        rows[cur]["smem"] = m.group(1)
for k, v in rows.items():
    if len(sys.argv) > 2 and sys.argv[2] not in k:
        continue
    print(f"{v.get('regs','?'):>4} regs  spill {v.get('spill','?'):>7}  smem {v.get('smem','0'):>6}  {k}")
if "error" in out:
    print(out)
