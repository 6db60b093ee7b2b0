"""fp64 CPU oracle for PackMamba's packed conv1d + selective scan (ctypes).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_2408_03865_b200`` (the CUDA product
path); neither imports the other.  The arithmetic lives in ``oracle.c``; this
module only marshals numpy arrays (converted exactly to fp64) into it.

Citations follow ``oracle.h``: P:n = PAPER.md line n, S:n = SPEC.md line n.
Parity pins: tests/test_oracle_*.py.  bf16 numerics of the GPU path are
"parity unpinned" beyond the stated tolerance.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_HDR = os.path.join(_HERE, "oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")

_f64p = ctypes.POINTER(ctypes.c_double)
_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (fp64, no fast-math, OpenMP over lanes)."""
    stale = (not os.path.exists(_LIB)) or any(
        os.path.getmtime(p) > os.path.getmtime(_LIB) for p in (_SRC, _HDR))
    if force or stale:
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
               "-Wall", "-Wextra", "-fno-fast-math", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True, cwd=_HERE)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.pmo_plan_fifo.argtypes = [_i32p, _i64, _i64, _i64p, _i64p, _i64p]
        L.pmo_plan_fifo.restype = ctypes.c_int
        L.pmo_plan_ffd.argtypes = [_i32p, _i64, _i64, _i64p, _i64p, _i64p]
        L.pmo_plan_ffd.restype = ctypes.c_int
        L.pmo_pack.argtypes = [_i32p, _i64, _i64, _i64p, _i64p, _u8p, _i64,
                               _u8p, _i32p, _i64]
        L.pmo_conv_fwd.argtypes = [_f64p, _f64p, _f64p, _i32p, _f64p,
                                   _i64, _i64, _i64, _i32, _i32]
        L.pmo_conv_bwd.argtypes = [_f64p, _f64p, _f64p, _i32p, _f64p,
                                   _f64p, _f64p, _f64p,
                                   _i64, _i64, _i64, _i32, _i32]
        L.pmo_scan_fwd.argtypes = [_f64p] * 7 + [_i32, _i32p, _f64p, _f64p,
                                                 _i64, _i64, _i64, _i32]
        L.pmo_scan_bwd_rows.argtypes = ([_f64p] * 7 + [_i32, _i32p, _f64p] +
                                        [_f64p] * 7 +
                                        [_i64, _i64, _i64, _i32, _i64, _i64])
        L.pmo_scan_fwd_eq3.argtypes = [_f64p] * 7 + [_i32, _i32p, _f64p,
                                                     _i64, _i64, _i64, _i32]
        L.pmo_seq_conv_fwd.argtypes = [_f64p, _f64p, _f64p, _f64p,
                                       _i64, _i64, _i32, _i32]
        L.pmo_seq_conv_bwd.argtypes = [_f64p] * 7 + [_i64, _i64, _i32, _i32]
        L.pmo_seq_scan_fwd.argtypes = [_f64p] * 7 + [_i32, _f64p,
                                                     _i64, _i64, _i32]
        L.pmo_seq_scan_bwd.argtypes = ([_f64p] * 7 + [_i32] + [_f64p] * 8 +
                                       [_i64, _i64, _i32])
        L.pmo_scan_fwd_ext.argtypes = ([_f64p] * 7 + [_i32, _i32, _i32p, _f64p, _f64p, _f64p, _f64p,
                                        _f64p,
                                        _i64, _i64, _i64, _i32])
        L.pmo_scan_bwd_ext.argtypes = ([_f64p] * 7 + [_i32, _i32, _i32p] + [_f64p] * 13 +
                                       [_i64, _i64, _i64, _i32])
        L.pmo_num_threads.restype = ctypes.c_int
        L.pmo_set_num_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


# ----------------------------------------------------------------------------
# marshalling helpers (no arithmetic)
# ----------------------------------------------------------------------------

def _f64(a):
    if a is None:
        return None
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a, t=_f64p):
    return None if a is None else a.ctypes.data_as(t)


def num_threads() -> int:
    return int(lib().pmo_num_threads())


def set_num_threads(n: int) -> None:
    lib().pmo_set_num_threads(int(n))


class CapacityError(ValueError):
    """A sequence is longer than the pack."""


def plan_fifo(lens, cap):
    """FIFO-seal plan.  Returns (seq_row, seq_off, n_rows)."""
    lens = np.ascontiguousarray(np.asarray(lens, dtype=np.int32))
    n = lens.shape[0]
    row = np.zeros(max(n, 1), np.int64)
    off = np.zeros(max(n, 1), np.int64)
    nr = np.zeros(1, np.int64)
    rc = lib().pmo_plan_fifo(_p(lens, _i32p), n, int(cap), _p(row, _i64p),
                             _p(off, _i64p), _p(nr, _i64p))
    if rc != 0:
        raise CapacityError("sequence exceeds pack capacity")
    return row[:n], off[:n], int(nr[0])


def plan_ffd(lens, cap):
    """First-fit-decreasing plan (P:273 local greedy)."""
    lens = np.ascontiguousarray(np.asarray(lens, dtype=np.int32))
    n = lens.shape[0]
    row = np.zeros(max(n, 1), np.int64)
    off = np.zeros(max(n, 1), np.int64)
    nr = np.zeros(1, np.int64)
    rc = lib().pmo_plan_ffd(_p(lens, _i32p), n, int(cap), _p(row, _i64p),
                            _p(off, _i64p), _p(nr, _i64p))
    if rc != 0:
        raise CapacityError("sequence exceeds pack capacity")
    return row[:n], off[:n], int(nr[0])


def pack(lens, cap, src_records, seq_row=None, seq_off=None):
    """Pack token-major records (Σlen, rec_bytes) uint8 -> (rows, cap, rec) + pos.

    Uses the FIFO plan unless a plan is given."""
    lens = np.ascontiguousarray(np.asarray(lens, dtype=np.int32))
    if seq_row is None:
        seq_row, seq_off, n_rows = plan_fifo(lens, cap)
    else:
        n_rows = int(np.max(seq_row)) + 1 if len(seq_row) else 0
    seq_row = np.ascontiguousarray(seq_row, dtype=np.int64)
    seq_off = np.ascontiguousarray(seq_off, dtype=np.int64)
    src = np.ascontiguousarray(src_records, dtype=np.uint8)
    rec = src.shape[1] if src.ndim == 2 else 1
    dst = np.empty((n_rows, cap, rec), np.uint8)
    pos = np.empty((n_rows, cap), np.int32)
    lib().pmo_pack(_p(lens, _i32p), lens.shape[0], int(cap), _p(seq_row, _i64p),
                   _p(seq_off, _i64p), _p(src, _u8p), rec, _p(dst, _u8p),
                   _p(pos, _i32p), n_rows)
    return dst, pos


def conv_fwd(x, w, bias, pos, silu=True):
    """Alg 1 conv1d_pack forward.  x (R,Dn,L); w (Dn,K); bias (Dn)|None."""
    x, w, bias = _f64(x), _f64(w), _f64(bias)
    pos = np.ascontiguousarray(pos, dtype=np.int32)
    R, Dn, L = x.shape
    K = w.shape[1]
    out = np.empty_like(x)
    lib().pmo_conv_fwd(_p(x), _p(w), _p(bias), _p(pos, _i32p), _p(out),
                       R, Dn, L, K, int(bool(silu)))
    return out


def conv_bwd(x, w, bias, pos, dout, silu=True):
    """Adjoint of conv_fwd -> (dx, dw, dbias)."""
    x, w, bias, dout = _f64(x), _f64(w), _f64(bias), _f64(dout)
    pos = np.ascontiguousarray(pos, dtype=np.int32)
    R, Dn, L = x.shape
    K = w.shape[1]
    dx = np.empty_like(x)
    dw = np.empty_like(w)
    db = np.empty(Dn, np.float64)
    lib().pmo_conv_bwd(_p(x), _p(w), _p(bias), _p(pos, _i32p), _p(dout),
                       _p(dx), _p(dw), _p(db), R, Dn, L, K, int(bool(silu)))
    return dx, dw, db


def scan_fwd(u, dt, A, B, C, D, dt_bias, pos, softplus=True, return_h=False):
    """ScanOp_pack forward (Alg 2; Eq 1a/1b/2a).  Returns y (and h if asked)."""
    u, dt, A, B, C = _f64(u), _f64(dt), _f64(A), _f64(B), _f64(C)
    D, dt_bias = _f64(D), _f64(dt_bias)
    pos = np.ascontiguousarray(pos, dtype=np.int32)
    R, Dn, L = u.shape
    N = A.shape[1]
    y = np.empty_like(u)
    h = np.empty((R, Dn, L, N), np.float64) if return_h else None
    lib().pmo_scan_fwd(_p(u), _p(dt), _p(A), _p(B), _p(C), _p(D), _p(dt_bias),
                       int(bool(softplus)), _p(pos, _i32p), _p(y), _p(h),
                       R, Dn, L, N)
    return (y, h) if return_h else y


def scan_bwd(u, dt, A, B, C, D, dt_bias, pos, dy, softplus=True, rows=None):
    """Adjoint of scan_fwd -> dict(du, ddt, dA, dB, dC, dD, ddt_bias).

    rows=(r0, r1) restricts the computation to a row subset (param grads are
    then sums over those rows only; du/ddt/dB/dC outside the subset are 0)."""
    u, dt, A, B, C = _f64(u), _f64(dt), _f64(A), _f64(B), _f64(C)
    D, dt_bias, dy = _f64(D), _f64(dt_bias), _f64(dy)
    pos = np.ascontiguousarray(pos, dtype=np.int32)
    R, Dn, L = u.shape
    N = A.shape[1]
    r0, r1 = (0, R) if rows is None else rows
    out = dict(du=np.zeros_like(u), ddt=np.zeros_like(u),
               dA=np.empty((Dn, N)), dB=np.zeros((R, N, L)),
               dC=np.zeros((R, N, L)), dD=np.empty(Dn), ddt_bias=np.empty(Dn))
    lib().pmo_scan_bwd_rows(
        _p(u), _p(dt), _p(A), _p(B), _p(C), _p(D), _p(dt_bias),
        int(bool(softplus)), _p(pos, _i32p), _p(dy),
        _p(out["du"]), _p(out["ddt"]), _p(out["dA"]), _p(out["dB"]),
        _p(out["dC"]), _p(out["dD"]), _p(out["ddt_bias"]),
        R, Dn, L, N, int(r0), int(r1))
    return out


def scan_fwd_eq3(u, dt, A, B, C, D, dt_bias, pos, softplus=True):
    """O3: Eq 3 brute force, O(L^2) -- tiny inputs only."""
    u, dt, A, B, C = _f64(u), _f64(dt), _f64(A), _f64(B), _f64(C)
    D, dt_bias = _f64(D), _f64(dt_bias)
    pos = np.ascontiguousarray(pos, dtype=np.int32)
    R, Dn, L = u.shape
    N = A.shape[1]
    y = np.empty_like(u)
    lib().pmo_scan_fwd_eq3(_p(u), _p(dt), _p(A), _p(B), _p(C), _p(D),
                           _p(dt_bias), int(bool(softplus)), _p(pos, _i32p),
                           _p(y), R, Dn, L, N)
    return y


# --- O2: per-sequence (unpacked) operators -----------------------------------

def seq_conv_fwd(x, w, bias, silu=True):
    x, w, bias = _f64(x), _f64(w), _f64(bias)
    Dn, Ls = x.shape
    out = np.empty_like(x)
    lib().pmo_seq_conv_fwd(_p(x), _p(w), _p(bias), _p(out), Dn, Ls,
                           w.shape[1], int(bool(silu)))
    return out


def seq_conv_bwd(x, w, bias, dout, dw_acc, db_acc, silu=True):
    """Returns dx; accumulates into dw_acc, db_acc (fp64 arrays)."""
    x, w, bias, dout = _f64(x), _f64(w), _f64(bias), _f64(dout)
    Dn, Ls = x.shape
    dx = np.empty_like(x)
    lib().pmo_seq_conv_bwd(_p(x), _p(w), _p(bias), _p(dout), _p(dx),
                           _p(dw_acc), _p(db_acc), Dn, Ls, w.shape[1],
                           int(bool(silu)))
    return dx


def seq_scan_fwd(u, dt, A, B, C, D, dt_bias, softplus=True):
    u, dt, A, B, C = _f64(u), _f64(dt), _f64(A), _f64(B), _f64(C)
    D, dt_bias = _f64(D), _f64(dt_bias)
    Dn, Ls = u.shape
    y = np.empty_like(u)
    lib().pmo_seq_scan_fwd(_p(u), _p(dt), _p(A), _p(B), _p(C), _p(D),
                           _p(dt_bias), int(bool(softplus)), _p(y), Dn, Ls,
                           A.shape[1])
    return y


def seq_scan_bwd(u, dt, A, B, C, D, dt_bias, dy, acc, softplus=True):
    """Returns (du, ddt, dB, dC); accumulates dA, dD, ddt_bias into acc."""
    u, dt, A, B, C = _f64(u), _f64(dt), _f64(A), _f64(B), _f64(C)
    D, dt_bias, dy = _f64(D), _f64(dt_bias), _f64(dy)
    Dn, Ls = u.shape
    N = A.shape[1]
    du, ddt = np.empty_like(u), np.empty_like(u)
    dB, dC = np.empty((N, Ls)), np.empty((N, Ls))
    lib().pmo_seq_scan_bwd(_p(u), _p(dt), _p(A), _p(B), _p(C), _p(D),
                           _p(dt_bias), int(bool(softplus)), _p(dy), _p(du),
                           _p(ddt), _p(acc["dA"]), _p(dB), _p(dC),
                           _p(acc["dD"]), _p(acc["ddt_bias"]), Dn, Ls, N)
    return du, ddt, dB, dC


# --- NEXT-1 / NEXT-2: gate and state passing ---------------------------------

def scan_fwd_ext(u, dt, A, B, C, D, dt_bias, pos, z=None, h0=None, softplus=True, zoh=False,
                 want_decay=False):
    """Returns (out, h_last): out = y * silu(z) (y if z is None); h0 (R,Dn,N)
    is the state entering t=0 when pos[r,0] != 0; zoh selects Eq 2b
     for B-bar instead of Euler."""
    u, dt, A, B, C = _f64(u), _f64(dt), _f64(A), _f64(B), _f64(C)
    D, dt_bias, z, h0 = _f64(D), _f64(dt_bias), _f64(z), _f64(h0)
    pos = np.ascontiguousarray(pos, dtype=np.int32)
    R, Dn, L = u.shape
    N = A.shape[1]
    out = np.empty_like(u)
    h_last = np.empty((R, Dn, N))
    decay = np.empty((R, Dn, N))
    lib().pmo_scan_fwd_ext(_p(u), _p(dt), _p(A), _p(B), _p(C), _p(D), _p(dt_bias),
                           int(bool(softplus)), int(bool(zoh)), _p(pos, _i32p), _p(z), _p(h0),
                           _p(out),
                           _p(h_last), _p(decay), R, Dn, L, N)
    if want_decay:
        return out, h_last, decay
    return out, h_last


def scan_bwd_ext(u, dt, A, B, C, D, dt_bias, pos, dout, z=None, h0=None, dh_last=None,
                 softplus=True, zoh=False):
    """Adjoint of scan_fwd_ext -> dict(du, ddt, dA, dB, dC, dD, ddt_bias, dz, dh0)."""
    u, dt, A, B, C = _f64(u), _f64(dt), _f64(A), _f64(B), _f64(C)
    D, dt_bias, z, h0 = _f64(D), _f64(dt_bias), _f64(z), _f64(h0)
    dout, dh_last = _f64(dout), _f64(dh_last)
    pos = np.ascontiguousarray(pos, dtype=np.int32)
    R, Dn, L = u.shape
    N = A.shape[1]
    o = dict(du=np.zeros_like(u), ddt=np.zeros_like(u), dA=np.empty((Dn, N)),
             dB=np.zeros((R, N, L)), dC=np.zeros((R, N, L)), dD=np.empty(Dn),
             ddt_bias=np.empty(Dn), dz=np.zeros_like(u) if z is not None else None,
             dh0=np.zeros((R, Dn, N)) if h0 is not None else None)
    lib().pmo_scan_bwd_ext(_p(u), _p(dt), _p(A), _p(B), _p(C), _p(D), _p(dt_bias),
                           int(bool(softplus)), int(bool(zoh)), _p(pos, _i32p), _p(z), _p(h0),
                           _p(dout),
                           _p(dh_last), _p(o["du"]), _p(o["ddt"]), _p(o["dA"]), _p(o["dB"]),
                           _p(o["dC"]), _p(o["dD"]), _p(o["ddt_bias"]), _p(o["dz"]),
                           _p(o["dh0"]), R, Dn, L, N)
    return o
