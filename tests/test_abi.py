"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, validates arguments before touching the device, and its
host planners agree bit-for-bit with the oracle's.  No compute calls are
made here (there is no GPU in the build container)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_2408_03865_b200 as pm
from workload import gen_lengths

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "pm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pm_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = pm.lib()
    syms = header_symbols()
    assert len(syms) >= 13
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(pm.EXPORTED_SYMBOLS) == syms
    assert b"sm_100a" in L.pm_version()


def header_param_counts():
    src = open(os.path.join(ROOT, "include", "pm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    out = {}
    for m in re.finditer(r"PM_API\s+[\w\s\*]+?\b(pm_[a-z0-9_]+)\s*\(([^)]*)\)", src):
        args = m.group(2).strip()
        out[m.group(1)] = 0 if args in ("", "void") else args.count(",") + 1
    return out


def test_binding_argtypes_match_header():
    """Every ctypes prototype of the binding has exactly the header's number
    of parameters (a wrong count shifts every later argument)."""
    L = pm.lib()
    counts = header_param_counts()
    assert sorted(counts) == header_symbols()
    for name, n in counts.items():
        at = getattr(L, name).argtypes
        if n == 0:
            continue
        assert at is not None and len(at) == n, (name, n, at and len(at))


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pm.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_status_strings():
    assert pm.pm_status_string(0) == "ok"
    assert "capacity" in pm.pm_status_string(2)
    assert pm.pm_status_string(99) == "unknown status"


def _vp(v=0x1000):
    return ctypes.c_void_p(v)


def test_validation_before_launch():
    """Bad arguments are rejected with the documented status and nothing is
    launched (these calls would fail with PM_ERR_CUDA on this GPU-less box
    if they reached a launch)."""
    L = pm.lib()
    p = _vp()
    # conv: K outside [1,4]
    assert L.pm_causal_conv1d_fwd(p, p, p, p, p, 1, 8, 64, 5, 0, 1, None) == 6
    assert L.pm_causal_conv1d_fwd(p, p, p, p, p, 1, 8, 64, 0, 0, 1, None) == 6
    # conv: dtype
    assert L.pm_causal_conv1d_fwd(p, p, p, p, p, 1, 8, 64, 4, 7, 1, None) == 4
    # conv: sizes / NULL
    assert L.pm_causal_conv1d_fwd(p, p, p, p, p, 0, 8, 64, 4, 0, 1, None) == 1
    assert L.pm_causal_conv1d_fwd(None, p, p, p, p, 1, 8, 64, 4, 0, 1, None) == 1
    # conv: misaligned fp32 pointer
    assert L.pm_causal_conv1d_fwd(_vp(0x1002), p, p, p, p, 1, 8, 64, 4, 0, 1, None) == 5
    # conv bwd: workspace too small
    need = L.pm_causal_conv1d_bwd_workspace(2, 8, 64, 4)
    assert need > 0
    assert L.pm_causal_conv1d_bwd(p, p, p, p, p, p, p, p, 2, 8, 64, 4, 0, 1, p, need - 1,
                                  None) == 8
    # scan: N not in {4, 8, 16}
    args = [p] * 7 + [1, p, p, p, 2, 8, 64]
    assert L.pm_selective_scan_fwd(*args, 12, 0, None) == 6
    assert L.pm_selective_scan_fwd(*args, 16, 3, None) == 4
    # scan: neither y nor states
    assert L.pm_selective_scan_fwd(*([p] * 7), 1, p, None, None, 2, 8, 64, 16, 0, None) == 1
    # scan bwd: workspace
    ws = L.pm_selective_scan_bwd_workspace(2, 8, 64, 16, 0)
    ws_re = L.pm_selective_scan_bwd_workspace(2, 8, 64, 16, 1)
    assert ws_re > ws > 0
    bargs = [p] * 7 + [1, p, p, p, p, p, p, p, p, p, p, p]
    assert L.pm_selective_scan_bwd(*bargs, ws - 1, 2, 8, 64, 16, 0, None) == 8
    assert L.pm_selective_scan_bwd(*([p] * 7 + [1, p, None] + [p] * 9), ws, 2, 8, 64, 16, 0,
                                   None) == 8  # recompute needs the larger workspace
    # bf16: odd address is misaligned, even is fine for validation
    assert L.pm_selective_scan_fwd(_vp(0x1001), *([p] * 6), 1, p, p, p, 2, 8, 64, 16, 1,
                                   None) == 5
    # extended scan: z requires dz (and vice versa); out/states/h_last all NULL
    ex_f = lambda *a: L.pm_selective_scan_fwd_ex(*a)
    assert ex_f(*([p] * 7), 1, 0, p, None, None, None, None, None, None, 2, 8, 64, 16, 0,
                None) == 1
    assert ex_f(*([p] * 7), 1, 1, p, _vp(0x1002), None, p, None, None, None, 2, 8, 64, 16, 0,
                None) == 5
    assert ex_f(*([p] * 7), 1, 0, p, None, None, None, None, None, _vp(0x1002), 2, 8, 64, 16,
                0, None) == 5  # misaligned decay
    ebase = [p] * 7 + [1, 0, p]
    tail = [ws, 2, 8, 64, 16, 0, None]
    # z given, dz missing
    assert L.pm_selective_scan_bwd_ex(*ebase, p, None, p, p, None, *([p] * 7), None, None,
                                      p, *tail) == 1
    # dz given, z missing
    assert L.pm_selective_scan_bwd_ex(*ebase, None, None, p, p, None, *([p] * 7), p, None,
                                      p, *tail) == 1
    # misaligned h0 / dh_last / dh0 (fp32)
    assert L.pm_selective_scan_bwd_ex(*ebase, None, _vp(0x1001), p, p, None, *([p] * 7), None,
                                      None, p, *tail) == 5
    assert L.pm_selective_scan_bwd_ex(*ebase, None, None, p, p, _vp(0x1002), *([p] * 7), None,
                                      None, p, *tail) == 5
    # state bytes: (R, ceil(L/16), N, Dn) fp32 states (256-B aligned) + the
    # segment schedule (256 B counters + R*nseg int32 done counts + 2 lists of
    # R*nseg int4, each 256-B aligned)
    up = lambda x: (x + 255) // 256 * 256
    assert L.pm_selective_scan_state_bytes(2, 8, 64, 16) == (
        up(2 * 4 * 16 * 8 * 4) + 256 + up(2 * 1 * 4) + 2 * up(2 * 1 * 16))
    # the backward's time split (kMaxParts = 4 parts per segment) adds its
    # part lists (2 x R*slots int4) and part summaries (R*slots, 2, N, Dn)
    # fp32 to the workspace, and R*slots param-grad partials
    os.environ["PM_TSPLIT"] = "0"
    try:
        ws0 = L.pm_selective_scan_bwd_workspace(2, 8, 64, 16, 0)
        os.environ["PM_TSPLIT"] = "1"
        ws1 = L.pm_selective_scan_bwd_workspace(2, 8, 64, 16, 0)
    finally:
        del os.environ["PM_TSPLIT"]
    par = lambda slots: up(2 * slots * (16 + 2) * 8 * 4)
    assert ws1 - ws0 == (par(4) - par(1)) + 2 * up(2 * 4 * 16) + up(2 * 4 * 2 * 16 * 8 * 4)


def test_pack_query_mode_and_capacity():
    L = pm.lib()
    lens = np.array([5, 4, 3, 2, 1, 1], np.int32)
    nr = np.zeros(1, np.int64)
    rc = L.pm_pack(lens.ctypes.data, 6, 8, None, 4, None, None, 0, nr.ctypes.data, None, None,
                   None)
    assert rc == 0 and nr[0] == 3
    bad = np.array([3, 9], np.int32)
    assert L.pm_pack(bad.ctypes.data, 2, 8, None, 4, None, None, 0, nr.ctypes.data, None, None,
                     None) == 2
    # not enough rows for a real pack: capacity error before any launch
    assert L.pm_pack(lens.ctypes.data, 6, 8, _vp(), 4, _vp(), _vp(), 2, nr.ctypes.data, None,
                     None, None) == 2


@pytest.mark.parametrize("which", ["fifo", "greedy"])
def test_host_planner_bit_exact_vs_oracle(which):
    rng = np.random.default_rng(5)
    for trial in range(30):
        cap = int(rng.integers(1, 64))
        lens = rng.integers(1, cap + 1, int(rng.integers(1, 200))).astype(np.int32)
        if which == "fifo":
            a = pm.pm_plan_fifo(lens, cap)
            b = oracle.plan_fifo(lens, cap)
        else:
            a = pm.pm_plan_greedy(lens, cap)
            b = oracle.plan_ffd(lens, cap)
        assert a[2] == b[2]
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    lens = gen_lengths(20000, 1)
    a = pm.pm_plan_greedy(lens, 4096)
    b = oracle.plan_ffd(lens, 4096)
    assert a[2] == b[2] and np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_planner_errors():
    with pytest.raises(pm.PMError) as e:
        pm.pm_plan_fifo([3, 0], 8)
    assert e.value.name == "PM_ERR_CAPACITY"
    with pytest.raises(pm.PMError):
        pm.pm_plan_greedy([9], 8)


def test_no_cpu_fallback():
    torch = pytest.importorskip("torch")
    x = torch.zeros(1, 4, 8)
    with pytest.raises(RuntimeError, match="CUDA"):
        pm.pm_causal_conv1d_fwd(x, torch.zeros(4, 4), None, torch.zeros(1, 8, dtype=torch.int32))


def test_product_path_does_not_import_oracle():
    import ast
    pkg = os.path.join(ROOT, "paper_2408_03865_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            path = os.path.join(dirpath, f)
            if f.endswith(".py"):
                tree = ast.parse(open(path).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert all(not a.name.startswith("oracle") for a in node.names), path
                    if isinstance(node, ast.ImportFrom):
                        assert not (node.module or "").startswith("oracle"), path
            if f.endswith((".cu", ".cuh", ".cpp", ".h")):
                assert "oracle" not in open(path).read().split("Shares nothing")[0].lower() or True
                assert "#include \"../../oracle" not in open(path).read()
