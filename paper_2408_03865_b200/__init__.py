"""PackMamba (arXiv 2408.03865) packed conv1d + selective scan on B200.

Thin ctypes binding over ``libpm.so`` (the C ABI in ``include/pm.h``).  Every
function here only marshals arguments -- tensor data pointers, sizes, the
current CUDA stream -- into the same-named C entry point; all computation
runs in the library's sm_100a kernels.  There is no CPU fallback: if the
library is missing or the tensors are not on a CUDA device, calls raise.

PyTorch is used for device memory, streams and process groups only.
"""
from __future__ import annotations

import ctypes
import os

__all__ = [
    "PMError", "lib", "pm_status_string", "pm_plan_fifo", "pm_plan_greedy",
    "pm_pack", "pm_pack_planned", "pm_causal_conv1d_fwd", "pm_causal_conv1d_bwd",
    "pm_causal_conv1d_bwd_workspace", "pm_selective_scan_state_bytes",
    "pm_selective_scan_fwd", "pm_selective_scan_bwd",
    "pm_selective_scan_bwd_workspace", "pm_selective_scan_fwd_ex", "pm_selective_scan_bwd_ex",
    "pm_selective_scan_fwd_bwd", "pm_scan_chain_fwd", "pm_scan_chain_bwd",
    "pm_selective_scan_fwd_fixup", "pm_selective_scan_dh0", "EXPORTED_SYMBOLS",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# PM_LIB: an alternative in-tree build (A/B experiments, tools/gpu_ab_lib.sh)
LIB_PATH = os.environ.get("PM_LIB") or os.path.join(_HERE, "libpm.so")

PM_F32, PM_BF16 = 0, 1
STATUS = {0: "PM_OK", 1: "PM_ERR_INVALID_ARG", 2: "PM_ERR_CAPACITY", 3: "PM_ERR_SHAPE",
          4: "PM_ERR_DTYPE", 5: "PM_ERR_ALIGN", 6: "PM_ERR_UNSUPPORTED", 7: "PM_ERR_CUDA",
          8: "PM_ERR_WORKSPACE"}

# every symbol include/pm.h declares (checked by tests/test_abi.py)
EXPORTED_SYMBOLS = [
    "pm_status_string", "pm_version", "pm_plan_fifo", "pm_plan_greedy", "pm_pack",
    "pm_pack_planned", "pm_causal_conv1d_fwd", "pm_causal_conv1d_bwd_workspace",
    "pm_causal_conv1d_bwd", "pm_selective_scan_state_bytes", "pm_selective_scan_fwd",
    "pm_selective_scan_bwd_workspace", "pm_selective_scan_bwd", "pm_selective_scan_fwd_ex",
    "pm_selective_scan_bwd_ex", "pm_selective_scan_fwd_bwd", "pm_scan_chain_fwd",
    "pm_scan_chain_bwd", "pm_selective_scan_fwd_fixup", "pm_selective_scan_dh0",
]


class PMError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        self.name = STATUS.get(code, str(code))
        super().__init__(f"{where}: {self.name} ({pm_status_string(code)})")


_vp, _i64, _i32, _sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
_lib = None


def lib():
    """Load libpm.so.  The in-tree library is (re)built first when it is
    missing or older than its sources (``_build.stale``); a PM_LIB variant is
    loaded as is."""
    global _lib
    if _lib is None:
        from . import _build
        if LIB_PATH == _build.LIB:
            _build.build()  # no-op unless missing or stale
        elif not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"PM_LIB={LIB_PATH} does not exist")
        L = ctypes.CDLL(LIB_PATH)
        L.pm_status_string.restype = ctypes.c_char_p
        L.pm_status_string.argtypes = [ctypes.c_int]
        L.pm_version.restype = ctypes.c_char_p
        for f in ("pm_plan_fifo", "pm_plan_greedy"):
            getattr(L, f).argtypes = [_vp, _i64, _i64, _vp, _vp, _vp]
        L.pm_pack.argtypes = [_vp, _i64, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _vp]
        L.pm_pack_planned.argtypes = [_vp, _i64, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _vp]
        L.pm_causal_conv1d_fwd.argtypes = [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i32,
                                           ctypes.c_int, _i32, _vp]
        L.pm_causal_conv1d_bwd_workspace.restype = _sz
        L.pm_causal_conv1d_bwd_workspace.argtypes = [_i64, _i64, _i64, _i32]
        L.pm_causal_conv1d_bwd.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64,
                                           _i64, _i32, ctypes.c_int, _i32, _vp, _sz, _vp]
        L.pm_selective_scan_state_bytes.restype = _sz
        L.pm_selective_scan_state_bytes.argtypes = [_i64, _i64, _i64, _i32]
        L.pm_selective_scan_fwd.argtypes = [_vp] * 7 + [_i32, _vp, _vp, _vp, _i64, _i64, _i64,
                                                       _i32, ctypes.c_int, _vp]
        L.pm_selective_scan_bwd_workspace.restype = _sz
        L.pm_selective_scan_bwd_workspace.argtypes = [_i64, _i64, _i64, _i32, _i32]
        L.pm_selective_scan_bwd.argtypes = ([_vp] * 7 + [_i32] + [_vp] * 10 + [_vp, _sz] +
                                            [_i64, _i64, _i64, _i32, ctypes.c_int, _vp])
        L.pm_selective_scan_fwd_ex.argtypes = ([_vp] * 7 + [_i32, _i32] + [_vp] * 7 +
                                               [_i64, _i64, _i64, _i32, ctypes.c_int, _vp])
        L.pm_selective_scan_bwd_ex.argtypes = ([_vp] * 7 + [_i32, _i32] + [_vp] * 15 + [_vp, _sz] +
                                               [_i64, _i64, _i64, _i32, ctypes.c_int, _vp])
        L.pm_selective_scan_fwd_bwd.argtypes = ([_vp] * 7 + [_i32, _i32] + [_vp] * 19 + [_sz] +
                                                [_i64, _i64, _i64, _i32, ctypes.c_int, _vp])
        L.pm_scan_chain_fwd.argtypes = [_vp] * 8 + [_i64, _i64, _i64, _i32, _vp]
        L.pm_scan_chain_bwd.argtypes = [_vp] * 8 + [_i64, _i64, _i64, _i32, _vp]
        L.pm_selective_scan_fwd_fixup.argtypes = ([_vp] * 4 + [_i32] + [_vp] * 5 +
                                                  [_i64, _i64, _i64, _i32, ctypes.c_int, _vp])
        L.pm_selective_scan_dh0.argtypes = ([_vp] * 4 + [_i32] + [_vp] * 4 +
                                            [_i64, _i64, _i64, _i32, ctypes.c_int, _vp])
        for f in EXPORTED_SYMBOLS:
            if f not in ("pm_status_string", "pm_version") and not f.endswith(
                    ("_workspace", "_bytes")):
                getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def pm_status_string(code: int) -> str:
    return lib().pm_status_string(int(code)).decode()


def _check(rc: int, where: str) -> None:
    if rc != 0:
        raise PMError(rc, where)


# ----------------------------------------------------------------------------
# marshalling helpers
# ----------------------------------------------------------------------------

def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(t):
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _io(t):
    import torch
    if t.dtype == torch.float32:
        return PM_F32
    if t.dtype == torch.bfloat16:
        return PM_BF16
    raise TypeError(f"unsupported I/O dtype {t.dtype} (float32 or bfloat16)")


def _dev(*ts):
    for t in ts:
        if t is not None:
            if not t.is_cuda:
                raise RuntimeError("libpm runs on CUDA tensors only (no CPU fallback)")
            if not t.is_contiguous():
                raise RuntimeError("libpm needs contiguous tensors")


def _want(t, name, dtype=None, shape=None):
    """Argument check before the C call (the C ABI only sees void pointers):
    dtype and shape of every tensor argument."""
    if t is None:
        return
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")


def _scan_args(u, dt, A, B, C, Dskip, dt_bias, pos, **tok):
    """Validate the scan's inputs; returns (R, Dn, L, N).  ``tok``: more
    per-token (R,Dn,L) tensors in the I/O dtype (z, dy, dout, ...)."""
    import torch
    if u.dim() != 3:
        raise ValueError(f"u: expected (R, Dn, L), got shape {tuple(u.shape)}")
    R, Dn, L = u.shape
    io = u.dtype
    _io(u)
    if A.dim() != 2 or A.shape[0] != Dn:
        raise ValueError(f"A: expected (Dn={Dn}, N), got shape {tuple(A.shape)}")
    N = A.shape[1]
    _want(A, "A", torch.float32)
    _want(dt, "dt", io, (R, Dn, L))
    _want(B, "B", io, (R, N, L))
    _want(C, "C", io, (R, N, L))
    _want(Dskip, "Dskip", torch.float32, (Dn,))
    _want(dt_bias, "dt_bias", torch.float32, (Dn,))
    _want(pos, "pos", torch.int32, (R, L))
    for k, v in tok.items():
        _want(v, k, io, (R, Dn, L))
    return R, Dn, L, N


def _conv_args(x, w, bias, pos, **tok):
    import torch
    if x.dim() != 3:
        raise ValueError(f"x: expected (R, Dn, L), got shape {tuple(x.shape)}")
    R, Dn, L = x.shape
    _io(x)
    if w.dim() != 2 or w.shape[0] != Dn:
        raise ValueError(f"w: expected (Dn={Dn}, K), got shape {tuple(w.shape)}")
    _want(w, "w", torch.float32)
    _want(bias, "bias", torch.float32, (Dn,))
    _want(pos, "pos", torch.int32, (R, L))
    for k, v in tok.items():
        _want(v, k, x.dtype, (R, Dn, L))
    return R, Dn, L, w.shape[1]


def _host_i32(a):
    import numpy as np
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(ctypes.c_void_p)


# ----------------------------------------------------------------------------
# packing
# ----------------------------------------------------------------------------

def pm_plan_fifo(seq_lens, pack_len):
    """FIFO-seal plan on the host -> (seq_row, seq_off, n_rows)."""
    return _plan("pm_plan_fifo", seq_lens, pack_len)


def pm_plan_greedy(seq_lens, pack_len):
    """First-fit-decreasing plan (P:273 'local greedy') -> (row, off, n_rows)."""
    return _plan("pm_plan_greedy", seq_lens, pack_len)


def _plan(name, seq_lens, pack_len):
    import numpy as np
    lens, lp = _host_i32(seq_lens)
    n = lens.shape[0]
    row = np.zeros(max(n, 1), np.int64)
    off = np.zeros(max(n, 1), np.int64)
    nr = np.zeros(1, np.int64)
    _check(getattr(lib(), name)(lp, n, int(pack_len), row.ctypes.data, off.ctypes.data,
                                nr.ctypes.data), name)
    return row[:n], off[:n], int(nr[0])


def pm_pack(seq_lens, pack_len, src, dst=None, pos=None, max_rows=None):
    """Pack token-major records ``src`` (sum(len), ...) on the GPU.

    Returns (dst, pos, seq_row, seq_off).  ``dst``/``pos`` are allocated when
    not given: dst (n_rows, pack_len, *src.shape[1:]) like src, pos int32."""
    import numpy as np
    import torch
    _dev(src)
    lens, lp = _host_i32(seq_lens)
    n = lens.shape[0]
    rec = src.element_size() * (src[0].numel() if src.dim() > 1 else 1)
    row = np.zeros(max(n, 1), np.int64)
    off = np.zeros(max(n, 1), np.int64)
    nr = np.zeros(1, np.int64)
    L = lib()
    if dst is None or pos is None:
        _check(L.pm_pack(lp, n, int(pack_len), None, rec, None, None, 0, nr.ctypes.data,
                         None, None, None), "pm_pack(query)")
        rows = int(nr[0])
        dst = torch.empty((rows, pack_len, *src.shape[1:]), dtype=src.dtype, device=src.device)
        pos = torch.empty((rows, pack_len), dtype=torch.int32, device=src.device)
    _dev(dst, pos)
    mr = dst.shape[0] if max_rows is None else int(max_rows)
    _check(L.pm_pack(lp, n, int(pack_len), _ptr(src), rec, _ptr(dst), _ptr(pos), mr,
                     nr.ctypes.data, row.ctypes.data, off.ctypes.data, _stream(src)), "pm_pack")
    return dst, pos, row[:n], off[:n]


def pm_pack_planned(seq_lens, pack_len, seq_row, seq_off, n_rows, src, dst, pos):
    import numpy as np
    _dev(src, dst, pos)
    lens, lp = _host_i32(seq_lens)
    row = np.ascontiguousarray(seq_row, dtype=np.int64)
    off = np.ascontiguousarray(seq_off, dtype=np.int64)
    rec = src.element_size() * (src[0].numel() if src.dim() > 1 else 1)
    _check(lib().pm_pack_planned(lp, lens.shape[0], int(pack_len), row.ctypes.data,
                                 off.ctypes.data, int(n_rows), _ptr(src), rec, _ptr(dst),
                                 _ptr(pos), _stream(src)), "pm_pack_planned")
    return dst, pos


# ----------------------------------------------------------------------------
# conv1d_pack
# ----------------------------------------------------------------------------

def pm_causal_conv1d_fwd(x, w, bias, pos, out=None, silu=True):
    """Alg 1 conv1d_pack forward: x (R,Dn,L) f32|bf16, w (Dn,K) f32, pos (R,L) i32."""
    import torch
    _dev(x, w, bias, pos)
    R, Dn, L, _ = _conv_args(x, w, bias, pos, out=out)
    out = torch.empty_like(x) if out is None else out
    _dev(out)
    _check(lib().pm_causal_conv1d_fwd(_ptr(x), _ptr(w), _ptr(bias), _ptr(pos), _ptr(out), R, Dn,
                                      L, w.shape[1], _io(x), int(bool(silu)), _stream(x)),
           "pm_causal_conv1d_fwd")
    return out


def pm_causal_conv1d_bwd_workspace(R, Dn, L, K):
    return int(lib().pm_causal_conv1d_bwd_workspace(R, Dn, L, K))


def pm_causal_conv1d_bwd(x, w, bias, pos, dout, dx=None, dw=None, dbias=None, silu=True,
                         workspace=None):
    """Adjoint of conv1d_pack -> (dx, dw, dbias)."""
    import torch
    _dev(x, w, bias, pos, dout)
    R, Dn, L, K = _conv_args(x, w, bias, pos, dout=dout, dx=dx)
    _want(dw, "dw", torch.float32, (Dn, K))
    _want(dbias, "dbias", torch.float32, (Dn,))
    dx = torch.empty_like(x) if dx is None else dx
    dw = torch.empty_like(w) if dw is None else dw
    if dbias is None and bias is not None:
        dbias = torch.empty_like(bias)
    need = pm_causal_conv1d_bwd_workspace(R, Dn, L, K)
    if workspace is None:
        workspace = torch.empty(need, dtype=torch.uint8, device=x.device)
    _dev(dx, dw, dbias, workspace)
    _check(lib().pm_causal_conv1d_bwd(_ptr(x), _ptr(w), _ptr(bias), _ptr(pos), _ptr(dout),
                                      _ptr(dx), _ptr(dw), _ptr(dbias), R, Dn, L, K, _io(x),
                                      int(bool(silu)), _ptr(workspace), workspace.numel(),
                                      _stream(x)), "pm_causal_conv1d_bwd")
    return dx, dw, dbias


# ----------------------------------------------------------------------------
# ScanOp_pack
# ----------------------------------------------------------------------------

def _states_ok(states, R, Dn, L, N):
    import torch
    if states is None:
        return
    _want(states, "states", torch.float32)
    if states.numel() * 4 < pm_selective_scan_state_bytes(R, Dn, L, N):
        raise ValueError("states: smaller than pm_selective_scan_state_bytes()")


def _grad_outs(o, R, Dn, L, N, io):
    """Check caller-supplied gradient outputs (dtype and shape)."""
    import torch
    f32 = torch.float32
    spec = dict(du=(io, (R, Dn, L)), ddt=(io, (R, Dn, L)), dz=(io, (R, Dn, L)),
                dA=(f32, (Dn, N)), dB=(f32, (R, N, L)), dC=(f32, (R, N, L)), dD=(f32, (Dn,)),
                ddt_bias=(f32, (Dn,)), dh0=(f32, (R, Dn, N)))
    for k, v in o.items():
        if k in spec:
            _want(v, k, *spec[k])


def pm_selective_scan_state_bytes(R, Dn, L, N):
    return int(lib().pm_selective_scan_state_bytes(R, Dn, L, N))


def pm_selective_scan_bwd_workspace(R, Dn, L, N, recompute_states=False):
    return int(lib().pm_selective_scan_bwd_workspace(R, Dn, L, N, int(bool(recompute_states))))


def pm_selective_scan_fwd(u, dt, A, B, C, Dskip, dt_bias, pos, y=None, states=None,
                          dt_softplus=True, want_states=True):
    """ScanOp_pack forward (Alg 2; Eq 1a/1b/2a).  Returns (y, states)."""
    import torch
    _dev(u, dt, A, B, C, Dskip, dt_bias, pos)
    R, Dn, L, N = _scan_args(u, dt, A, B, C, Dskip, dt_bias, pos, y=y)
    y = torch.empty_like(u) if y is None else y
    if states is None and want_states:
        nb = pm_selective_scan_state_bytes(R, Dn, L, N)
        states = torch.empty(nb // 4, dtype=torch.float32, device=u.device)
    _dev(y, states)
    _check(lib().pm_selective_scan_fwd(_ptr(u), _ptr(dt), _ptr(A), _ptr(B), _ptr(C),
                                       _ptr(Dskip), _ptr(dt_bias), int(bool(dt_softplus)),
                                       _ptr(pos), _ptr(y), _ptr(states), R, Dn, L, N, _io(u),
                                       _stream(u)), "pm_selective_scan_fwd")
    return y, states


def pm_selective_scan_bwd(u, dt, A, B, C, Dskip, dt_bias, pos, dy, states=None,
                          dt_softplus=True, out=None, workspace=None):
    """Adjoint of ScanOp_pack.  Returns dict du, ddt, dA, dB, dC, dD, ddt_bias.

    ``out`` may supply preallocated outputs (same keys)."""
    import torch
    _dev(u, dt, A, B, C, Dskip, dt_bias, pos, dy, states)
    R, Dn, L, N = _scan_args(u, dt, A, B, C, Dskip, dt_bias, pos, dy=dy)
    _states_ok(states, R, Dn, L, N)
    o = dict(out or {})
    _grad_outs(o, R, Dn, L, N, u.dtype)
    dev = u.device
    f32 = dict(dtype=torch.float32, device=dev)
    o.setdefault("du", torch.empty_like(u))
    o.setdefault("ddt", torch.empty_like(u))
    o.setdefault("dA", torch.empty((Dn, N), **f32))
    o.setdefault("dB", torch.empty((R, N, L), **f32))
    o.setdefault("dC", torch.empty((R, N, L), **f32))
    o.setdefault("dD", torch.empty((Dn,), **f32) if Dskip is not None else None)
    o.setdefault("ddt_bias", torch.empty((Dn,), **f32) if dt_bias is not None else None)
    need = pm_selective_scan_bwd_workspace(R, Dn, L, N, states is None)
    if workspace is None:
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)
    _dev(workspace, *[v for v in o.values() if v is not None])
    _check(lib().pm_selective_scan_bwd(
        _ptr(u), _ptr(dt), _ptr(A), _ptr(B), _ptr(C), _ptr(Dskip), _ptr(dt_bias),
        int(bool(dt_softplus)), _ptr(pos), _ptr(states), _ptr(dy), _ptr(o["du"]), _ptr(o["ddt"]),
        _ptr(o["dA"]), _ptr(o["dB"]), _ptr(o["dC"]), _ptr(o["dD"]), _ptr(o["ddt_bias"]),
        _ptr(workspace), workspace.numel(), R, Dn, L, N, _io(u), _stream(u)),
        "pm_selective_scan_bwd")
    return o


def pm_selective_scan_fwd_ex(u, dt, A, B, C, Dskip, dt_bias, pos, z=None, h0=None, out=None,
                             states=None, h_last=None, dt_softplus=True, want_states=True,
                             want_last_state=False, zoh=False, decay=None, want_decay=False):
    """Extended ScanOp_pack forward: fused gate ``out = y * silu(z)`` (SURVEY
    NEXT-1) and cross-row state passing ``h0 -> h_last`` (NEXT-2, the
    paper's future work P:275); ``zoh`` selects Eq 2b's B-bar (NEXT-4)
    instead of Euler.  ``decay`` (R,Dn,N) receives d h_last / d h0 (the row
    summary of a context-parallel scan).  Returns (out, states, h_last), plus
    decay when want_decay."""
    import torch
    _dev(u, dt, A, B, C, Dskip, dt_bias, pos, z, h0)
    R, Dn, L, N = _scan_args(u, dt, A, B, C, Dskip, dt_bias, pos, z=z, out=out)
    for k, v in (("h0", h0), ("h_last", h_last), ("decay", decay)):
        _want(v, k, torch.float32, (R, Dn, N))
    out = torch.empty_like(u) if out is None else out
    if states is None and want_states:
        nb = pm_selective_scan_state_bytes(R, Dn, L, N)
        states = torch.empty(nb // 4, dtype=torch.float32, device=u.device)
    if h_last is None and want_last_state:
        h_last = torch.empty((R, Dn, N), dtype=torch.float32, device=u.device)
    if decay is None and want_decay:
        decay = torch.empty((R, Dn, N), dtype=torch.float32, device=u.device)
    _dev(out, states, h_last, decay)
    _check(lib().pm_selective_scan_fwd_ex(
        _ptr(u), _ptr(dt), _ptr(A), _ptr(B), _ptr(C), _ptr(Dskip), _ptr(dt_bias),
        int(bool(dt_softplus)), int(bool(zoh)), _ptr(pos), _ptr(z), _ptr(h0), _ptr(out),
        _ptr(states),
        _ptr(h_last), _ptr(decay), R, Dn, L, N, _io(u), _stream(u)), "pm_selective_scan_fwd_ex")
    if want_decay:
        return out, states, h_last, decay
    return out, states, h_last


def pm_selective_scan_bwd_ex(u, dt, A, B, C, Dskip, dt_bias, pos, dout, z=None, h0=None,
                             states=None, dh_last=None, dt_softplus=True, out=None,
                             workspace=None, want_dh0=None, zoh=False):
    """Adjoint of pm_selective_scan_fwd_ex.  Returns dict du, ddt, dA, dB, dC,
    dD, ddt_bias, dz (when z is given), dh0 (when h0 is given or want_dh0)."""
    import torch
    _dev(u, dt, A, B, C, Dskip, dt_bias, pos, dout, z, h0, states, dh_last)
    R, Dn, L, N = _scan_args(u, dt, A, B, C, Dskip, dt_bias, pos, dout=dout, z=z)
    for k, v in (("h0", h0), ("dh_last", dh_last)):
        _want(v, k, torch.float32, (R, Dn, N))
    _states_ok(states, R, Dn, L, N)
    o = dict(out or {})
    _grad_outs(o, R, Dn, L, N, u.dtype)
    dev = u.device
    f32 = dict(dtype=torch.float32, device=dev)
    o.setdefault("du", torch.empty_like(u))
    o.setdefault("ddt", torch.empty_like(u))
    o.setdefault("dA", torch.empty((Dn, N), **f32))
    o.setdefault("dB", torch.empty((R, N, L), **f32))
    o.setdefault("dC", torch.empty((R, N, L), **f32))
    o.setdefault("dD", torch.empty((Dn,), **f32) if Dskip is not None else None)
    o.setdefault("ddt_bias", torch.empty((Dn,), **f32) if dt_bias is not None else None)
    o.setdefault("dz", torch.empty_like(u) if z is not None else None)
    if want_dh0 is None:
        want_dh0 = h0 is not None
    o.setdefault("dh0", torch.empty((R, Dn, N), **f32) if want_dh0 else None)
    need = pm_selective_scan_bwd_workspace(R, Dn, L, N, states is None)
    if workspace is None:
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)
    _dev(workspace, *[v for v in o.values() if v is not None])
    _check(lib().pm_selective_scan_bwd_ex(
        _ptr(u), _ptr(dt), _ptr(A), _ptr(B), _ptr(C), _ptr(Dskip), _ptr(dt_bias),
        int(bool(dt_softplus)), int(bool(zoh)), _ptr(pos), _ptr(z), _ptr(h0), _ptr(states),
        _ptr(dout),
        _ptr(dh_last), _ptr(o["du"]), _ptr(o["ddt"]), _ptr(o["dA"]), _ptr(o["dB"]),
        _ptr(o["dC"]), _ptr(o["dD"]), _ptr(o["ddt_bias"]), _ptr(o["dz"]), _ptr(o["dh0"]),
        _ptr(workspace), workspace.numel(), R, Dn, L, N, _io(u), _stream(u)),
        "pm_selective_scan_bwd_ex")
    return o


def pm_selective_scan_fwd_bwd(u, dt, A, B, C, Dskip, dt_bias, pos, dout, states, z=None,
                              h0=None, out=None, h_last=None, decay=None, dh_last=None,
                              dt_softplus=True, zoh=False, grads=None, workspace=None,
                              want_dh0=None):
    """Forward + backward in one call (pm.h: the backward launched
    programmatically behind the library's own forward).  ``states`` is
    required (pm_selective_scan_state_bytes); ``out``/``h_last``/``decay``
    are optional forward outputs.  Returns (out, grads) with grads the dict
    of pm_selective_scan_bwd_ex."""
    import torch
    _dev(u, dt, A, B, C, Dskip, dt_bias, pos, dout, z, h0, states, dh_last, out, h_last, decay)
    R, Dn, L, N = _scan_args(u, dt, A, B, C, Dskip, dt_bias, pos, dout=dout, z=z, out=out)
    for k, v in (("h0", h0), ("dh_last", dh_last), ("h_last", h_last), ("decay", decay)):
        _want(v, k, torch.float32, (R, Dn, N))
    if states is None:
        raise ValueError("states is required")
    _states_ok(states, R, Dn, L, N)
    o = dict(grads or {})
    _grad_outs(o, R, Dn, L, N, u.dtype)
    dev = u.device
    f32 = dict(dtype=torch.float32, device=dev)
    o.setdefault("du", torch.empty_like(u))
    o.setdefault("ddt", torch.empty_like(u))
    o.setdefault("dA", torch.empty((Dn, N), **f32))
    o.setdefault("dB", torch.empty((R, N, L), **f32))
    o.setdefault("dC", torch.empty((R, N, L), **f32))
    o.setdefault("dD", torch.empty((Dn,), **f32) if Dskip is not None else None)
    o.setdefault("ddt_bias", torch.empty((Dn,), **f32) if dt_bias is not None else None)
    o.setdefault("dz", torch.empty_like(u) if z is not None else None)
    if want_dh0 is None:
        want_dh0 = h0 is not None
    o.setdefault("dh0", torch.empty((R, Dn, N), **f32) if want_dh0 else None)
    need = pm_selective_scan_bwd_workspace(R, Dn, L, N, False)
    if workspace is None:
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)
    _dev(workspace, *[v for v in o.values() if v is not None])
    _check(lib().pm_selective_scan_fwd_bwd(
        _ptr(u), _ptr(dt), _ptr(A), _ptr(B), _ptr(C), _ptr(Dskip), _ptr(dt_bias),
        int(bool(dt_softplus)), int(bool(zoh)), _ptr(pos), _ptr(z), _ptr(h0), _ptr(out),
        _ptr(states), _ptr(h_last), _ptr(decay), _ptr(dout), _ptr(dh_last), _ptr(o["du"]),
        _ptr(o["ddt"]), _ptr(o["dA"]), _ptr(o["dB"]), _ptr(o["dC"]), _ptr(o["dD"]),
        _ptr(o["ddt_bias"]), _ptr(o["dz"]), _ptr(o["dh0"]), _ptr(workspace), workspace.numel(),
        R, Dn, L, N, _io(u), _stream(u)), "pm_selective_scan_fwd_bwd")
    return out, o


# ----------------------------------------------------------------------------
# context-parallel scan pieces (NEXT-2); composed in .cp
# ----------------------------------------------------------------------------

def _rdn(R, Dn, N, dev):
    import torch
    return torch.empty((R, Dn, N), dtype=torch.float32, device=dev)


def pm_scan_chain_fwd(decay, h_last_local, pos=None, cont=None, h_init=None, h_in=None,
                      h_last=None, chain_decay=None):
    """Compose row summaries along the chains (pm.h) -> (h_in, h_last, chain_decay)."""
    import torch
    R, Dn, N = decay.shape
    _dev(decay, h_last_local, pos, cont, h_init)
    for k, v in (("decay", decay), ("h_last_local", h_last_local)):
        _want(v, k, torch.float32, (R, Dn, N))
    _want(h_init, "h_init", torch.float32, (Dn, N))
    _want(pos, "pos", torch.int32)
    _want(cont, "cont", torch.int32, (R,))
    if pos is not None and (pos.dim() != 2 or pos.shape[0] != R):
        raise ValueError(f"pos: expected ({R}, L), got shape {tuple(pos.shape)}")
    L = pos.shape[1] if pos is not None else 0
    h_in = _rdn(R, Dn, N, decay.device) if h_in is None else h_in
    h_last = _rdn(R, Dn, N, decay.device) if h_last is None else h_last
    if chain_decay is None:
        chain_decay = torch.empty((Dn, N), dtype=torch.float32, device=decay.device)
    _dev(h_in, h_last, chain_decay)
    _check(lib().pm_scan_chain_fwd(_ptr(pos), _ptr(cont), _ptr(decay), _ptr(h_last_local),
                                   _ptr(h_init), _ptr(h_in), _ptr(h_last), _ptr(chain_decay), R,
                                   Dn, L, N, _stream(decay)), "pm_scan_chain_fwd")
    return h_in, h_last, chain_decay


def pm_scan_chain_bwd(decay, dh0_local, pos=None, cont=None, dh_last_ext=None, g_end=None,
                      dh_last=None, dh_init=None):
    """Compose the cotangents of every row's h_last (pm.h) -> (dh_last, dh_init)."""
    import torch
    R, Dn, N = decay.shape
    _dev(decay, dh0_local, pos, cont, dh_last_ext, g_end)
    for k, v in (("decay", decay), ("dh0_local", dh0_local), ("dh_last_ext", dh_last_ext)):
        _want(v, k, torch.float32, (R, Dn, N))
    _want(g_end, "g_end", torch.float32, (Dn, N))
    _want(pos, "pos", torch.int32)
    _want(cont, "cont", torch.int32, (R,))
    L = pos.shape[1] if pos is not None else 0
    dh_last = _rdn(R, Dn, N, decay.device) if dh_last is None else dh_last
    if dh_init is None:
        dh_init = torch.empty((Dn, N), dtype=torch.float32, device=decay.device)
    _dev(dh_last, dh_init)
    _check(lib().pm_scan_chain_bwd(_ptr(pos), _ptr(cont), _ptr(decay), _ptr(dh0_local),
                                   _ptr(dh_last_ext), _ptr(g_end), _ptr(dh_last), _ptr(dh_init),
                                   R, Dn, L, N, _stream(decay)), "pm_scan_chain_bwd")
    return dh_last, dh_init


def pm_selective_scan_fwd_fixup(dt, A, C, dt_bias, pos, h_in, out, states=None, z=None,
                                dt_softplus=True):
    """Correct ``out`` (and ``states``) in place over the continuing prefixes (pm.h)."""
    import torch
    _dev(dt, A, C, dt_bias, pos, h_in, out, states, z)
    R, Dn, L, N = _scan_args(out, dt, A, C, C, None, dt_bias, pos, z=z)
    _want(h_in, "h_in", torch.float32, (R, Dn, N))
    _states_ok(states, R, Dn, L, N)
    _check(lib().pm_selective_scan_fwd_fixup(
        _ptr(dt), _ptr(A), _ptr(C), _ptr(dt_bias), int(bool(dt_softplus)), _ptr(pos), _ptr(z),
        _ptr(h_in), _ptr(out), _ptr(states), R, Dn, L, N, _io(out), _stream(out)),
        "pm_selective_scan_fwd_fixup")
    return out


def pm_selective_scan_dh0(dt, A, C, dt_bias, pos, dout, z=None, dh0_local=None,
                          dt_softplus=True):
    """Each row's dLoss/dh0 through its own outputs (pm.h) -> dh0_local (R,Dn,N)."""
    _dev(dt, A, C, dt_bias, pos, dout, z)
    R, Dn, L, N = _scan_args(dout, dt, A, C, C, None, dt_bias, pos, z=z)
    dh0_local = _rdn(R, Dn, N, dout.device) if dh0_local is None else dh0_local
    _dev(dh0_local)
    _check(lib().pm_selective_scan_dh0(
        _ptr(dt), _ptr(A), _ptr(C), _ptr(dt_bias), int(bool(dt_softplus)), _ptr(pos), _ptr(z),
        _ptr(dout), _ptr(dh0_local), R, Dn, L, N, _io(dout), _stream(dout)),
        "pm_selective_scan_dh0")
    return dh0_local
