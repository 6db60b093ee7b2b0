"""Multi-process (world_size 2, gloo, CPU) test of the data-parallel plumbing
of the hot path (paper_2408_03865_b200.dp): row sharding + one all-reduce of
the flattened parameter gradients ("8-GPU data parallel").

The per-rank gradients come from the fp64 oracle (test infrastructure); the
check is that the all-reduced [dA | dD | ddt_bias | dw | db] equals the
single-process gradients of all rows, and that per-row outputs do not depend
on the number of ranks (rows are seeded by global row id)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _grads_for_rows(cfg, rows_g, rows_layout_all):
    import oracle
    import workload
    layout = [rows_layout_all[r] for r in rows_g]
    pos, valid = workload.pos_from_rows(layout, cfg.L)
    T = workload.row_tensors(torch, cfg, rows_g, valid, device="cpu", dtype=torch.float32)
    P = {k: v.double().numpy() for k, v in workload.params(torch, cfg).items()}
    f = {k: v.double().numpy() for k, v in T.items()}
    u = oracle.conv_fwd(f["x"], P["w"], P["bias"], pos)
    g = oracle.scan_bwd(u, f["dt"], P["A"], f["B"], f["C"], P["D"], P["dt_bias"], pos, f["dy"])
    dx, dw, db = oracle.conv_bwd(f["x"], P["w"], P["bias"], pos, g["du"])
    y = oracle.scan_fwd(u, f["dt"], P["A"], f["B"], f["C"], P["D"], P["dt_bias"], pos)
    return dict(dA=g["dA"], dD=g["dD"], ddt_bias=g["ddt_bias"], dw=dw, db=db), y


def _worker(rank, world, port, cfg, layout, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2408_03865_b200.dp import ParamGrads, shard_rows
    rows = list(shard_rows(cfg.R * world, rank, world))
    grads, y = _grads_for_rows(cfg, rows, layout)
    pg = ParamGrads(torch, cfg.Dn, cfg.N, cfg.K, "cpu")
    for k, v in grads.items():
        pg[k].copy_(torch.as_tensor(v, dtype=torch.float32))
    pg.allreduce(dist)
    q.put((rank, {k: pg[k].numpy().copy() for k in grads}, rows, y))
    dist.barrier()
    dist.destroy_process_group()


def test_row_shards():
    from paper_2408_03865_b200.dp import shard_rows
    assert list(shard_rows(8, 0, 2)) == [0, 1, 2, 3]
    assert list(shard_rows(8, 1, 2)) == [4, 5, 6, 7]
    assert sum(len(shard_rows(64, r, 8)) for r in range(8)) == 64
    with pytest.raises(ValueError):
        shard_rows(6, 0, 4)


def test_allreduce_param_grads_world2():
    import workload
    cfg = workload.Shape("dp", 2, 48, 6, 4, 4, "f32")  # 2 rows per rank
    world = 2
    rng = np.random.default_rng(0)
    layout = []
    for _ in range(cfg.R * world):
        lens, t = [], 0
        while True:
            ln = int(rng.integers(1, 20))
            if t + ln > cfg.L:
                break
            lens.append(ln)
            t += ln
        layout.append(lens)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, layout, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref, yref = _grads_for_rows(cfg, list(range(cfg.R * world)), layout)
    for rank, got, rows, y in res:
        for k in ref:
            np.testing.assert_allclose(got[k], ref[k], rtol=2e-6, atol=1e-6, err_msg=k)
        # per-row outputs are independent of the sharding (seeded by global row)
        np.testing.assert_array_equal(y, yref[rows[0]:rows[-1] + 1])
