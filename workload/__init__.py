"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NO arithmetic of the method (no packing plan, no conv, no
scan): it only draws random numbers and builds position arrays from explicit
per-row layouts.  Both sides (``oracle`` and ``paper_2408_03865_b200``) may
consume it; it imports neither.

Recipe, following the paper's
workload "sequences ranging in length from 57 to 2048, with an average length
of 646" packed into rows of 4096:

* lengths: truncated lognormal on [57, 2048], sigma = 1.0, mu = 6.3547
  (fitted so the mean is ~646);
* x ~ N(0,1); dt ~ N(0, 0.5^2); dt_bias = softplus^-1(exp(U[ln 1e-3, ln 1e-1]));
  A[d,n] = -(n+1) * exp(N(0, 0.1^2)); B, C ~ N(0,1); D = 1 + N(0, 0.1^2);
  w, bias ~ U(-0.5, 0.5); dy ~ N(0,1);
* padding slots hold x = 0 and dy = 0 (reading Q8).

Every per-row tensor is drawn row by row from a generator seeded by
(config, tensor name, GLOBAL row id), so row r is identical for any number of
GPUs the rows are sharded over.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

# Paper workload constants and the fitted lognormal.
LEN_MIN, LEN_MAX, LEN_MU, LEN_SIGMA = 57, 2048, 6.3547, 1.0


def seed_of(*parts) -> int:
    """Stable 63-bit seed from arbitrary parts (config, tensor, row, ...)."""
    h = hashlib.sha256("/".join(str(p) for p in parts).encode()).digest()
    return int.from_bytes(h[:8], "little") & ((1 << 63) - 1)


def gen_lengths(n: int, seed: int, lo: int = LEN_MIN, hi: int = LEN_MAX,
                mu: float = LEN_MU, sigma: float = LEN_SIGMA) -> np.ndarray:
    """n lengths from a lognormal truncated to [lo, hi] (rejection sampling)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = np.empty(0, np.int64)
    while out.shape[0] < n:
        draw = np.rint(rng.lognormal(mu, sigma, size=2 * n + 16)).astype(np.int64)
        draw = draw[(draw >= lo) & (draw <= hi)]
        out = np.concatenate([out, draw])
    return out[:n].astype(np.int32)


def pos_from_rows(rows, L: int) -> tuple[np.ndarray, np.ndarray]:
    """Build (pos, valid) of shape (R, L) from an explicit layout.

    ``rows[r]`` is the list of sequence lengths laid out left to right in row
    r; the rest of the row is padding.  pos runs 0..len-1 inside a sequence
    and is 0 on padding (the PackedBatch invariants); ``valid`` is
    True on sequence slots and False on padding."""
    R = len(rows)
    pos = np.zeros((R, L), np.int32)
    valid = np.zeros((R, L), bool)
    for r, lens in enumerate(rows):
        t = 0
        for ln in lens:
            assert ln >= 1 and t + ln <= L, "layout does not fit the row"
            pos[r, t:t + ln] = np.arange(ln, dtype=np.int32)
            valid[r, t:t + ln] = True
            t += ln
    return pos, valid


def rows_from_plan(lens, seq_row, seq_off, n_rows):
    """Turn a plan (row, offset per sequence) into per-row length lists."""
    rows = [[] for _ in range(n_rows)]
    order = np.lexsort((np.asarray(seq_off), np.asarray(seq_row)))
    for i in order:
        rows[int(seq_row[i])].append(int(lens[i]))
    return rows


@dataclass
class Shape:
    """One workload shape (BASELINE.json configs)."""
    name: str
    R: int
    L: int
    Dn: int
    N: int
    K: int
    dtype: str  # "f32" | "bf16" (I/O dtype of the per-token tensors)
    layout: str = "lognormal"  # "lognormal" | "explicit"
    rows: list = field(default_factory=list)  # explicit layouts


# BASELINE.json "configs" (index = configs[i]); C2/C4 rows proposed in SURVEY §8(d)
CONFIGS = {
    "tiny": Shape("tiny", 1, 64, 16, 4, 4, "f32", "explicit", [[20, 30, 14]]),
    "130m": Shape("130m", 8, 2048, 1536, 16, 4, "f32"),
    "1.4b": Shape("1.4b", 8, 4096, 4096, 16, 4, "bf16"),
    "2.8b": Shape("2.8b", 8, 4096, 5120, 16, 4, "bf16"),
    "2.8b-16k": Shape("2.8b-16k", 64, 16384, 5120, 16, 4, "bf16"),
}


def lengths_stream(cfg_name: str, n: int) -> np.ndarray:
    """The length sequence a config's rows are filled from (seed per config)."""
    return gen_lengths(n, seed_of(cfg_name, "lengths"))


# ----------------------------------------------------------------------------
# value tensors (torch; generated row by row on the target device)
# ----------------------------------------------------------------------------

def _gen(torch, device, *parts):
    g = torch.Generator(device=device)
    g.manual_seed(seed_of(*parts))
    return g


def params(torch, cfg: Shape, device="cpu", seed_tag="p"):
    """Parameters: A (Dn,N), D, dt_bias (Dn), w (Dn,K), bias (Dn), fp32."""
    Dn, N, K = cfg.Dn, cfg.N, cfg.K
    f = dict(device=device, dtype=torch.float32)
    g = _gen(torch, device, cfg.name, seed_tag, "A")
    A = -(torch.arange(1, N + 1, **f)[None, :]) * torch.exp(
        0.1 * torch.randn(Dn, N, generator=g, **f))
    g = _gen(torch, device, cfg.name, seed_tag, "D")
    D = 1.0 + 0.1 * torch.randn(Dn, generator=g, **f)
    g = _gen(torch, device, cfg.name, seed_tag, "dt_bias")
    target = torch.exp(torch.empty(Dn, **f).uniform_(np.log(1e-3), np.log(1e-1),
                                                     generator=g))
    dt_bias = target + torch.log(-torch.expm1(-target))  # softplus^-1
    g = _gen(torch, device, cfg.name, seed_tag, "w")
    w = torch.empty(Dn, K, **f).uniform_(-0.5, 0.5, generator=g)
    g = _gen(torch, device, cfg.name, seed_tag, "bias")
    bias = torch.empty(Dn, **f).uniform_(-0.5, 0.5, generator=g)
    return dict(A=A, D=D, dt_bias=dt_bias, w=w, bias=bias)


def row_tensors(torch, cfg: Shape, rows_global, valid, device="cpu",
                dtype=None, seed_tag="x"):
    """Per-token tensors x, dt, dy (R,Dn,L) and B, C (R,N,L) for the given
    GLOBAL row ids.  ``valid`` (len(rows_global), L) bool marks sequence
    slots; x and dy are zero on padding."""
    dtype = dtype or (torch.bfloat16 if cfg.dtype == "bf16" else torch.float32)
    R, Dn, N, L = len(rows_global), cfg.Dn, cfg.N, cfg.L
    f = dict(device=device, dtype=torch.float32)
    out = {k: torch.empty((R, Dn, L), device=device, dtype=dtype)
           for k in ("x", "dt", "dy")}
    out.update({k: torch.empty((R, N, L), device=device, dtype=dtype)
                for k in ("B", "C")})
    vmask = torch.as_tensor(np.asarray(valid), device=device)
    for i, r in enumerate(rows_global):
        m = vmask[i].to(torch.float32)
        for name, scale, shape, masked in (("x", 1.0, (Dn, L), True),
                                           ("dt", 0.5, (Dn, L), False),
                                           ("dy", 1.0, (Dn, L), True),
                                           ("B", 1.0, (N, L), False),
                                           ("C", 1.0, (N, L), False)):
            g = _gen(torch, device, cfg.name, seed_tag, name, int(r))
            v = scale * torch.randn(shape, generator=g, **f)
            if masked:
                v = v * m[None, :]
            out[name][i].copy_(v.to(dtype))
    return out
