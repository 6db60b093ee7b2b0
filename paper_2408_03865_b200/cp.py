"""Context-parallel selective scan over cut sequences (
the paper's future work: "cut long sequences into multiple parts and
pass the hidden state between these parts ... parallel strategies for
infinitely long sequences").

A sequence longer than a pack continues from row r-1 into row r when
pos[r, 0] != 0; rows may also continue across ranks (rank k's first row
continues rank k-1's last row).  Every step runs in libpm's kernels (pm.h,
"Context-parallel scan"); this module only sequences the calls and, across
GPUs, exchanges one (Dn, N) summary pair per rank with all_gather:

forward   local pass (h0 = 0) -> per-row (decay, h_last_local)
          -> pm_scan_chain_fwd (within the rank; across ranks on the gathered
             (chain_decay, h_last[R-1]) of every rank) -> h_in per row
          -> pm_selective_scan_fwd_fixup: out and the chunk states corrected
             over each continuing row's prefix only;
backward  pm_selective_scan_dh0 (each row's dLoss/dh0 through its own outputs)
          -> pm_scan_chain_bwd (within the rank; across ranks on the gathered
             (chain_decay, dh_init)) -> the cotangent of every row's h_last
          -> pm_selective_scan_bwd_ex(h0 = h_in, dh_last = that cotangent).

torch.distributed is plumbing only (NCCL on the GPU box; gloo in tests).
"""
from __future__ import annotations

from dataclasses import dataclass

from . import (pm_scan_chain_bwd, pm_scan_chain_fwd, pm_selective_scan_bwd_ex,
               pm_selective_scan_dh0, pm_selective_scan_fwd_ex, pm_selective_scan_fwd_fixup)


@dataclass
class CPContext:
    """What the backward needs from the forward."""
    states: object       # chunk states of the TRUE sequence (fixed up)
    h_in: object         # (R, Dn, N) state entering every row
    h_last: object       # (R, Dn, N) true state after every row
    decay: object        # (R, Dn, N) d h_last / d h0 per row
    chain_decay: object  # (Dn, N) d h_last[R-1] / d h_init of this rank


def _gather(dist, group, t):
    """all_gather of one (Dn, N) summary -> (world, Dn, N), rank order."""
    import torch
    world = dist.get_world_size(group)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t.contiguous(), group=group)
    return torch.stack(out)


def _ones(torch, n, dev):
    return torch.ones(n, dtype=torch.int32, device=dev)


def scan_fwd_cp(u, dt, A, B, C, D, dt_bias, pos, z=None, h_init=None, dist=None, group=None,
                dt_softplus=True, zoh=False):
    """Forward of the rows of this rank, with sequences cut across rows (and
    ranks).  h_init (Dn, N): the state entering the first row of rank 0 (the
    same tensor on every rank, or None = 0).  Returns (out, CPContext)."""
    import torch
    R, Dn, L = u.shape
    N = A.shape[1]
    zero = torch.zeros((R, Dn, N), dtype=torch.float32, device=u.device)
    out, states, hll, decay = pm_selective_scan_fwd_ex(
        u, dt, A, B, C, D, dt_bias, pos, z=z, h0=zero, want_last_state=True, want_decay=True,
        dt_softplus=dt_softplus, zoh=zoh)
    multi = dist is not None and dist.get_world_size(group) > 1
    # across ranks the summary E_k must be taken with h_init_k = 0 (the
    # global h_init enters once, through the chain over the ranks)
    h_in, h_last, cd = pm_scan_chain_fwd(decay, hll, pos=pos, h_init=None if multi else h_init)
    if multi:
        # rank k: h_last[R-1] = chain_decay_k * h_init_k + E_k (E_k: with h_init_k = 0)
        k = _rank(dist, group)
        Ds, Es = _gather(dist, group, cd), _gather(dist, group, h_last[R - 1])
        W = Ds.shape[0]
        hin_ranks, _, _ = pm_scan_chain_fwd(Ds, Es, cont=_ones(torch, W, u.device),
                                            h_init=h_init)
        h_in, h_last, cd = pm_scan_chain_fwd(decay, hll, pos=pos, h_init=hin_ranks[k],
                                             h_in=h_in, h_last=h_last, chain_decay=cd)
    pm_selective_scan_fwd_fixup(dt, A, C, dt_bias, pos, h_in, out, states=states, z=z,
                                dt_softplus=dt_softplus)
    return out, CPContext(states, h_in, h_last, decay, cd)


def scan_bwd_cp(u, dt, A, B, C, D, dt_bias, pos, dout, ctx, z=None, dh_last=None, dist=None,
                group=None, dt_softplus=True, zoh=False):
    """Backward of scan_fwd_cp.  dh_last (R, Dn, N) or None: external
    cotangents of the rows' final states (e.g. of the last part).  Returns the
    dict of pm_selective_scan_bwd_ex plus dh_init = dLoss/dh_init (on rank 0;
    param grads are this rank's partial sums, all-reduced by the caller)."""
    import torch
    dh0l = pm_selective_scan_dh0(dt, A, C, dt_bias, pos, dout, z=z, dt_softplus=dt_softplus)
    G, dh_init = pm_scan_chain_bwd(ctx.decay, dh0l, pos=pos, dh_last_ext=dh_last)
    if dist is not None and dist.get_world_size(group) > 1:
        # rank k: dh_init_k = chain_decay_k * g_end_k + E'_k (E'_k: with g_end_k = 0);
        # g_end_k = dh_init_{k+1}: a backward chain over the ranks
        k = _rank(dist, group)
        Ds, Eps = _gather(dist, group, ctx.chain_decay), _gather(dist, group, dh_init)
        W = Ds.shape[0]
        G_ranks, dh_init_all = pm_scan_chain_bwd(Ds, Eps, cont=_ones(torch, W, u.device))
        G, dh_init = pm_scan_chain_bwd(ctx.decay, dh0l, pos=pos, dh_last_ext=dh_last,
                                       g_end=G_ranks[k], dh_last=G, dh_init=dh_init)
        dh_init = dh_init_all  # (the chain over ranks' entry cotangent)
    g = pm_selective_scan_bwd_ex(u, dt, A, B, C, D, dt_bias, pos, dout, z=z, h0=ctx.h_in,
                                 states=ctx.states, dh_last=G, dt_softplus=dt_softplus, zoh=zoh)
    g["dh_init"] = dh_init
    return g


def _rank(dist, group):
    return 0 if dist is None else dist.get_rank(group)
