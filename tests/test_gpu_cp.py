"""Context-parallel scan on the GPU: sequences
cut over several rows (and over two ranks), forward and backward through
paper_2408_03865_b200.cp (local pass -> chain composition -> prefix fix-up;
dh0 summary -> backward chain -> backward), against the fp64 oracle run on
the UNCUT sequences (all rows laid end to end as one row: every cut is a
continuation, every other row start a head)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import oracle  # noqa: E402
import paper_2408_03865_b200 as pm  # noqa: E402
from paper_2408_03865_b200 import cp  # noqa: E402
import workload  # noqa: E402
from tests._common import TOL, rel_err, to_np  # noqa: E402

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DT = {"f32": torch.float32, "bf16": torch.bfloat16}


def layout(R, L, full=3, start=1000):
    """Row 0 continues an external state (pos starts at `start`); that
    sequence runs through rows 0..full-1 and 100 slots of row `full`, which
    then holds two short sequences; row full+1 is a fresh sequence cut into
    row full+2 (60 slots) followed by padding; later rows are single
    sequences."""
    assert R >= full + 3 and L >= 256
    pos = np.zeros((R, L), np.int32)
    valid = np.ones((R, L), bool)
    t = start
    for r in range(full):
        pos[r] = np.arange(t, t + L)
        t += L
    pos[full, :100] = np.arange(t, t + 100)
    pos[full, 100:160] = np.arange(60)
    pos[full, 160:] = np.arange(L - 160)
    pos[full + 1] = np.arange(L)
    pos[full + 2, :60] = np.arange(L, L + 60)
    pos[full + 2, 60:] = 0  # padding: each slot its own sequence (reading Q8)
    valid[full + 2, 60:] = False
    for r in range(full + 3, R):
        pos[r] = np.arange(L)
    return pos, valid


def problem(R, Dn, L, N, io, seed, gate, full=3):
    pos_np, valid = layout(R, L, full)
    shape = workload.Shape(f"cp{seed}", R, L, Dn, N, 4, io)
    T = workload.row_tensors(torch, shape, list(range(R)), valid, device="cuda", dtype=DT[io])
    P = workload.params(torch, shape, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(seed)
    u = torch.randn((R, Dn, L), device="cuda", generator=g).to(DT[io])
    z = torch.randn((R, Dn, L), device="cuda", generator=g).to(DT[io]) if gate else None
    h_init = 0.5 * torch.randn((Dn, N), device="cuda", generator=g)
    dh_last = torch.zeros((R, Dn, N), device="cuda")
    dh_last[R - 1] = torch.randn((Dn, N), device="cuda", generator=g)
    return torch.as_tensor(pos_np, device="cuda"), u, z, T, P, h_init, dh_last


def uncut_oracle(pos, u, z, T, P, h_init, dh_last):
    """All rows laid end to end as ONE row (h0 = h_init, dh_last of the last
    row) -- the uncut sequences."""
    cat = lambda t: None if t is None else np.concatenate(list(to_np(t)), axis=-1)[None]
    pos1 = np.concatenate(list(to_np(pos).astype(np.int32)), axis=-1)[None]
    args = (cat(u), cat(T["dt"]), to_np(P["A"]), cat(T["B"]), cat(T["C"]), to_np(P["D"]),
            to_np(P["dt_bias"]), pos1)
    out, hl = oracle.scan_fwd_ext(*args, z=cat(z), h0=to_np(h_init)[None])
    g = oracle.scan_bwd_ext(*args, cat(T["dy"]), z=cat(z), h0=to_np(h_init)[None],
                            dh_last=to_np(dh_last[-1])[None])
    return out, hl, g


def cat_rows(t):
    return np.concatenate(list(to_np(t)), axis=-1)[None]


@pytest.mark.parametrize("io", ["f32", "bf16"])
@pytest.mark.parametrize("gate", [False, True])
def test_cut_sequences_match_uncut_oracle(io, gate):
    R, Dn, L, N = 7, 64, 256, 16
    pos, u, z, T, P, h_init, dh_last = problem(R, Dn, L, N, io, seed=5 + gate, gate=gate)
    args = (u, T["dt"], P["A"], T["B"], T["C"], P["D"], P["dt_bias"], pos)
    out, ctx = cp.scan_fwd_cp(*args, z=z, h_init=h_init)
    g = cp.scan_bwd_cp(*args, T["dy"], ctx, z=z, dh_last=dh_last)
    torch.cuda.synchronize()
    ro, rhl, rg = uncut_oracle(pos, u, z, T, P, h_init, dh_last)
    tf, tb = TOL[(io, "fwd")], TOL[(io, "bwd")]
    assert rel_err(cat_rows(out), ro) <= tf
    assert rel_err(to_np(ctx.h_last)[-1], rhl[0]) <= tf
    for k in ("du", "ddt", "dB", "dC") + (("dz",) if gate else ()):
        e = rel_err(cat_rows(g[k]), rg[k])
        assert e <= tb, (k, e)
    for k in ("dA", "dD", "ddt_bias"):
        e = rel_err(to_np(g[k]), rg[k])
        assert e <= tb, (k, e)
    assert rel_err(to_np(g["dh_init"]), rg["dh0"][0]) <= tb


def test_fixup_touches_only_continuing_prefixes():
    """The fix-up changes out only on the slots before each continuing row's
    first head: rows that start a sequence and every slot after a head keep
    the local pass's values bit for bit."""
    R, Dn, L, N = 7, 64, 256, 16
    pos, u, z, T, P, h_init, _ = problem(R, Dn, L, N, "f32", seed=9, gate=False)
    args = (u, T["dt"], P["A"], T["B"], T["C"], P["D"], P["dt_bias"], pos)
    zero = torch.zeros((R, Dn, N), device="cuda")
    local, _, _ = pm.pm_selective_scan_fwd_ex(*args, h0=zero, want_last_state=True)
    out, _ = cp.scan_fwd_cp(*args, h_init=h_init)
    torch.cuda.synchronize()
    p = to_np(pos)
    for r in range(R):
        heads = np.nonzero(p[r] == 0)[0]
        fh = int(heads[0]) if p[r, 0] != 0 and heads.size else (L if p[r, 0] != 0 else 0)
        assert torch.equal(out[r, :, fh:], local[r, :, fh:]), r
        if fh > 0:
            assert not torch.equal(out[r, :, :fh], local[r, :, :fh]), r


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cp_rank(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    R, Dn, L, N = 8, 64, 256, 16
    pos, u, z, T, P, h_init, dh_last = problem(R, Dn, L, N, "f32", seed=21, gate=True, full=4)
    rows = slice(rank * R // world, (rank + 1) * R // world)
    sl = lambda t: None if t is None else t[rows].contiguous()
    Tl = {k: sl(v) for k, v in T.items()}
    args = (sl(u), Tl["dt"], P["A"], Tl["B"], Tl["C"], P["D"], P["dt_bias"], sl(pos))
    out, ctx = cp.scan_fwd_cp(*args, z=sl(z), h_init=h_init, dist=dist)
    g = cp.scan_bwd_cp(*args, Tl["dy"], ctx, z=sl(z), dh_last=sl(dh_last), dist=dist)
    for k in ("dA", "dD", "ddt_bias"):
        dist.all_reduce(g[k])
    torch.cuda.synchronize()
    q.put((rank, out.cpu().numpy(), {k: v.cpu().numpy() for k, v in g.items() if v is not None}))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_chain_across_the_rank_boundary():
    """8 rows over 2 ranks (rank 0: rows 0-3, rank 1: rows 4-7): the sequence
    entering row 0 from h_init runs through rows 0-3 into 100 slots of row 4,
    i.e. across the rank boundary; rows 5/6 hold another cut sequence inside
    rank 1.  The gathered per-rank summaries compose the state entering rank
    1 (forward) and the cotangent leaving rank 0 (backward); the results
    match the uncut oracle."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cp_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    R, Dn, L, N = 8, 64, 256, 16
    pos, u, z, T, P, h_init, dh_last = problem(R, Dn, L, N, "f32", seed=21, gate=True, full=4)
    ro, _, rg = uncut_oracle(pos, u, z, T, P, h_init, dh_last)
    cat_np = lambda a: np.concatenate(list(a), axis=-1)[None]
    out = np.concatenate([r[1] for r in res], 0)
    assert rel_err(cat_np(out), ro) <= TOL[("f32", "fwd")]
    for k in ("du", "ddt", "dB", "dC", "dz"):
        got = np.concatenate([r[2][k] for r in res], 0)
        e = rel_err(cat_np(got), rg[k])
        assert e <= TOL[("f32", "bwd")], (k, e)
    for k in ("dA", "dD", "ddt_bias"):
        assert rel_err(res[0][2][k], rg[k]) <= TOL[("f32", "bwd")], k
    assert rel_err(res[0][2]["dh_init"], rg["dh0"][0]) <= TOL[("f32", "bwd")]
