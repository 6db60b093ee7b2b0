"""Build libpm.so (sm_100a) in-tree with nvcc.  No JIT cache: the .so lives
next to this file so it travels with the repo snapshot to the GPU box."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpm.so")
SOURCES = ["pack.cu", "conv.cu", "scan.cu", "scan_fwd.cu", "scan_bwd.cu", "scan_bwd2.cu", "cp.cu", "tsplit.cu"]
HEADERS = ["common.cuh", "scan_impl.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "-I", os.path.join(ROOT, "include")]


def _inputs():
    files = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    files.append(os.path.join(ROOT, "include", "pm.h"))
    files.append(os.path.abspath(__file__))
    return files


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _inputs())


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False,
          out: str = LIB, defines: tuple = ()) -> str:
    """Build libpm.so; `out`/`defines` build a variant (e.g. out=libpm_b.so,
    defines=("PM_FWD_POLY=0",)) for A/B experiments loaded through PM_LIB."""
    if out == LIB and not defines and not force and not stale():
        return LIB
    objs = []
    bdir = os.path.join(HERE, "build" if out == LIB else "build_" + os.path.basename(out)[:-3])
    os.makedirs(bdir, exist_ok=True)
    procs = []
    for s in SOURCES:
        o = os.path.join(bdir, s.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, s), "-o", o]
        if ptxas_v:
            cmd += ["-Xptxas", "-v"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT), s))
        objs.append(o)
    failed = False
    for p, s in procs:
        log, _ = p.communicate()
        if p.returncode != 0 or (ptxas_v and log):
            sys.stderr.write(log.decode())
        failed |= p.returncode != 0
    if failed:
        raise RuntimeError("nvcc failed")
    tmp = out + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "shared", "-o", tmp, *objs,
           "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    # python _build.py [--force] [-v] [--out libpm_x.so] [-DNAME=V ...]
    a = sys.argv[1:]
    out = os.path.join(HERE, a[a.index("--out") + 1]) if "--out" in a else LIB
    defs = tuple(x[2:] for x in a if x.startswith("-D"))
    print(build(force="--force" in a, verbose=True, ptxas_v="-v" in a, out=out, defines=defs))
