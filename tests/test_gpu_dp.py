"""Data-parallel path on the GPU ("8-GPU data
parallel"): two ranks (processes) on one GPU, each running libpm's four
kernels on its shard of the packed rows and all-reducing the flat
parameter-gradient buffer [dA | dD | ddt_bias | dw | db] (gloo here: the
driver's GPU box has one GPU; NCCL is the same call on the 8-GPU box).

Checks: the all-reduced buffer equals the single-rank run over all rows
(one launch of every kernel over the whole batch) up to fp32 summation
order, and every rank's per-token outputs of its rows are bit-identical to
the same rows of the single-rank run (rows are independent, seeded by global
row id, and a kernel's per-row arithmetic does not depend on the other rows
of its launch)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg():
    import workload
    return workload.Shape("dp-gpu", 4, 2048, 512, 16, 4, "bf16")  # 4 rows per rank


def _layout(cfg, total):
    import oracle
    import workload
    n = total * cfg.L // 300 + 64
    lens = workload.lengths_stream(cfg.name, n)
    row, off, nr = oracle.plan_fifo(lens, cfg.L)
    assert nr - 1 >= total
    keep = row < total
    return workload.rows_from_plan(lens[keep], row[keep], off[keep], total)


def _run_rows(cfg, rows_g, layout):
    """The bench's step on the given global rows (one launch per kernel)."""
    import paper_2408_03865_b200 as pm
    import workload
    from paper_2408_03865_b200.dp import ParamGrads
    pos_np, valid = workload.pos_from_rows([layout[r] for r in rows_g], cfg.L)
    pos = torch.as_tensor(pos_np, device="cuda")
    T = workload.row_tensors(torch, cfg, rows_g, valid, device="cuda")
    P = workload.params(torch, cfg, device="cuda")
    pg = ParamGrads(torch, cfg.Dn, cfg.N, cfg.K, "cuda")
    R, L, Dn, N = len(rows_g), cfg.L, cfg.Dn, cfg.N
    u = pm.pm_causal_conv1d_fwd(T["x"], P["w"], P["bias"], pos)
    st = torch.empty(pm.pm_selective_scan_state_bytes(R, Dn, L, N) // 4, dtype=torch.float32,
                     device="cuda")
    y = torch.empty_like(u)
    _, g = pm.pm_selective_scan_fwd_bwd(u, T["dt"], P["A"], T["B"], T["C"], P["D"], P["dt_bias"],
                                        pos, T["dy"], st, out=y,
                                        grads=dict(dA=pg["dA"], dD=pg["dD"],
                                                   ddt_bias=pg["ddt_bias"]))
    dx, _, _ = pm.pm_causal_conv1d_bwd(T["x"], P["w"], P["bias"], pos, g["du"], dw=pg["dw"],
                                       dbias=pg["db"])
    torch.cuda.synchronize()
    return pg, dict(u=u, y=y, dx=dx, du=g["du"], ddt=g["ddt"], dB=g["dB"], dC=g["dC"])


def _worker(rank, world, port, layout, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2408_03865_b200.dp import shard_rows
    cfg = _cfg()
    rows = list(shard_rows(cfg.R * world, rank, world))
    pg, out = _run_rows(cfg, rows, layout)
    pg.allreduce(dist)
    torch.cuda.synchronize()
    # numpy (pickled by value): torch tensors would be shared through file
    # descriptors that vanish when this process exits
    q.put((rank, rows, pg.flat.cpu().numpy().copy(),
           {k: v.float().cpu().numpy() for k, v in out.items()}))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_libpm_allreduce_matches_single_rank():
    cfg = _cfg()
    layout = _layout(cfg, cfg.R * WORLD)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, layout, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    pg1, out1 = _run_rows(cfg, list(range(cfg.R * WORLD)), layout)
    ref = pg1.flat.cpu().numpy().astype(np.float64)
    rms = float(np.sqrt(np.mean(ref * ref)))
    for rank, rows, flat, out in sorted(res, key=lambda t: t[0]):
        # fp32 sums of the same terms in another grouping (per-rank partials)
        err = np.max(np.abs(flat - ref) / (np.abs(ref) + rms))
        assert err <= 1e-5, (rank, err)
        for k, v in out.items():
            ref1 = out1[k][rows[0]:rows[-1] + 1].float().cpu().numpy()
            assert np.array_equal(v, ref1), (rank, k)
