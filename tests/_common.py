"""Shared test helpers: tolerance metric (reading Q14) and seeded
problem construction from ``workload`` (no method arithmetic here)."""
from __future__ import annotations

import numpy as np

# north_star tolerances (BASELINE.json): fp32 fwd 1e-4, fp32 grads 1e-3,
# bf16 I/O with fp32 accumulation 2e-2.
TOL = {("f32", "fwd"): 1e-4, ("f32", "bwd"): 1e-3,
       ("bf16", "fwd"): 2e-2, ("bf16", "bwd"): 2e-2}


def rel_err(got, ref) -> float:
    """max_i |g_i - r_i| / (|r_i| + rms(r))  (reading Q14)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    if ref.size == 0:
        return 0.0
    rms = float(np.sqrt(np.mean(ref * ref)))
    den = np.abs(ref) + (rms if rms > 0 else 1e-300)
    return float(np.max(np.abs(got - ref) / den))


def to_np(t):
    """Exact fp64 copy of a torch tensor (bf16 -> fp32 -> fp64 is exact)."""
    import torch
    if t is None:
        return None
    return t.detach().to(torch.float64).cpu().numpy()


def layout(kind: str, R: int, L: int, rng) -> list:
    """Per-row sequence-length layouts, including the stress layouts of
    SURVEY §8(d)."""
    rows = []
    for r in range(R):
        if kind == "one":            # one sequence per row
            rows.append([L])
        elif kind == "heads":        # every slot a head
            rows.append([1] * L)
        elif kind == "random":       # random lengths, some padding
            lens, t = [], 0
            while True:
                ln = int(rng.integers(1, max(2, L // 3)))
                if t + ln > L:
                    break
                lens.append(ln)
                t += ln
            rows.append(lens)
        elif kind == "short":        # length-1/2/3 sequences mixed with longer
            lens, t = [], 0
            while True:
                ln = int(rng.choice([1, 1, 2, 3, 17, 40]))
                if t + ln > L:
                    break
                lens.append(ln)
                t += ln
            rows.append(lens)
        elif kind == "edges":        # heads at 16k-1, 16k, 16k+1, 64k, 8k+-1
            cuts = sorted({c for k in range(1, L // 8 + 1)
                           for c in (16 * k - 1, 16 * k, 16 * k + 1, 64 * k, 8 * k - 1, 8 * k + 1)
                           if 0 < c < L})
            cuts = [c for i, c in enumerate(cuts) if i % 3 != 2]
            b = [0] + cuts + [L]
            rows.append([b[i + 1] - b[i] for i in range(len(b) - 1)])
        else:
            raise ValueError(kind)
    return rows
