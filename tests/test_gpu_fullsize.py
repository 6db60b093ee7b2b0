"""Full-size parity at BASELINE.json shapes, in the launch configuration
bench.py times (all rows of a GPU in one launch of each kernel).

The fp64 oracle cannot run every row in seconds, so each test samples rows:
the per-token outputs of a sampled row from the FULL launch are compared
element by element with the oracle fed that row's exact GPU inputs; the
parameter gradients (sums over all rows) are checked (a) on a single-row
launch against the oracle and (b) on the full launch through properties
that hold at any size (dD = sum dy*u; dbias = sum dpre recomputed in fp64)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import paper_2408_03865_b200 as pm
import workload
from tests._common import TOL, rel_err, to_np

pytestmark = pytest.mark.gpu


def build(cfg, R=None, seed_rows=None):
    R = R or cfg.R
    n = int(R * cfg.L / 500) + 64
    while True:
        lens = workload.lengths_stream(cfg.name, n)
        row, off, nr = oracle.plan_fifo(lens, cfg.L)
        if nr - 1 >= R:
            break
        n *= 2
    keep = row < R
    rows = workload.rows_from_plan(lens[keep], row[keep], off[keep], R)
    pos_np, valid = workload.pos_from_rows(rows, cfg.L)
    shape = workload.Shape(cfg.name, R, cfg.L, cfg.Dn, cfg.N, cfg.K, cfg.dtype)
    T = workload.row_tensors(torch, shape, list(range(R)), valid, device="cuda")
    P = workload.params(torch, shape, device="cuda")
    return pos_np, valid, T, P


def chain(pos, T, P):
    """The bench's step: conv fwd, the fused scan fwd+bwd call, conv bwd."""
    u = pm.pm_causal_conv1d_fwd(T["x"], P["w"], P["bias"], pos)
    R, Dn, L = u.shape
    st = torch.empty(pm.pm_selective_scan_state_bytes(R, Dn, L, P["A"].shape[1]) // 4,
                     dtype=torch.float32, device="cuda")
    y = torch.empty_like(u)
    _, g = pm.pm_selective_scan_fwd_bwd(u, T["dt"], P["A"], T["B"], T["C"], P["D"], P["dt_bias"],
                                        pos, T["dy"], st, out=y)
    del st
    dx, dw, db = pm.pm_causal_conv1d_bwd(T["x"], P["w"], P["bias"], pos, g["du"])
    torch.cuda.synchronize()
    return dict(u=u, y=y, dx=dx, dw=dw, db=db, **g)


def row_np(t, r):
    return to_np(t[r:r + 1])


def fwd_split_env(cfg, R):
    """The forward's lane split the library picks for a launch of R rows
    (scan_impl.cuh fwd_throughput_bound), as a PM_FWD_SPLIT value that pins
    the same choice on a launch of fewer rows (the backward's time split,
    PM_TSPLIT, follows the same test: on iff latency-bound)."""
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    load = R * cfg.L * ((cfg.Dn + 127) // 128) / (nsm * 4)
    return "1" if 10 * load >= 3 * cfg.L else "4"


# Every BASELINE.json config at its full size, in the launch configuration
# bench.py times (all rows of one GPU in one launch): 130m (fp32, latency-
# bound: 4-lane split forward, serialized backward), 1.4b and 2.8b (bf16,
# 8 x 4096), 2.8b-16k (bf16, all 64 rows x 16384 on one GPU).
@pytest.mark.parametrize("name", ["130m", "1.4b", "2.8b", "2.8b-16k"])
def test_fullsize_sampled_rows(monkeypatch, name):
    cfg = workload.CONFIGS[name]
    R = cfg.R
    io = cfg.dtype
    pos_np, valid, T, P = build(cfg, R)
    pos = torch.as_tensor(pos_np, device="cuda")
    out = chain(pos, T, P)
    p = {k: to_np(v) for k, v in P.items()}
    # (a) sampled rows of the full launch (first, middle, last -- the last
    # ends in padding), every per-token output element by element
    for r in sorted({0, R // 2, R - 1}):
        pr = pos_np[r:r + 1]
        x = row_np(T["x"], r)
        ru = oracle.conv_fwd(x, p["w"], p["bias"], pr)
        assert rel_err(row_np(out["u"], r), ru) <= TOL[(io, "fwd")], (r, "u")
        u = row_np(out["u"], r)
        args = (u, row_np(T["dt"], r), p["A"], row_np(T["B"], r), row_np(T["C"], r), p["D"],
                p["dt_bias"], pr)
        e = rel_err(row_np(out["y"], r), oracle.scan_fwd(*args))
        assert e <= TOL[(io, "fwd")], (r, "y", e)
        g = oracle.scan_bwd(*args, row_np(T["dy"], r))
        for k in ("du", "ddt", "dB", "dC"):
            e = rel_err(row_np(out[k], r), g[k])
            assert e <= TOL[(io, "bwd")], (r, k, e)
        rdx, _, _ = oracle.conv_bwd(x, p["w"], p["bias"], pr, row_np(out["du"], r))
        assert rel_err(row_np(out["dx"], r), rdx) <= TOL[(io, "bwd")], (r, "dx")
        del g, args, u, x
    # (b) properties of the full launch's parameter gradients, any size:
    # dD[d] = sum_{r,t} dy u (fp64 from the launch's own tensors)
    dD = sum((T["dy"][i].double() * out["u"][i].double()).sum(dim=1) for i in range(R))
    dD = dD.cpu().numpy()
    assert rel_err(to_np(out["dD"]), dD) <= TOL[(io, "bwd")]
    # (c) the parameter gradients of one row's launch vs the oracle, in the
    # full launch's shape (the forward's lane split pinned to the full
    # launch's choice so the row's outputs must match it bit for bit)
    r = R - 1
    monkeypatch.setenv("PM_FWD_SPLIT", fwd_split_env(cfg, R))
    monkeypatch.setenv("PM_TSPLIT", "0" if fwd_split_env(cfg, R) == "1" else "1")
    T1 = {k: v[r:r + 1].contiguous() for k, v in T.items()}
    o1 = chain(pos[r:r + 1].contiguous(), T1, P)
    for k in ("du", "ddt", "dB", "dC", "y", "u", "dx"):  # same row, other rows absent
        assert torch.equal(o1[k][0], out[k][r]), k
    del out
    pr = pos_np[r:r + 1]
    x = row_np(T["x"], r)
    args = (row_np(o1["u"], 0), row_np(T["dt"], r), p["A"], row_np(T["B"], r),
            row_np(T["C"], r), p["D"], p["dt_bias"], pr)
    g = oracle.scan_bwd(*args, row_np(T["dy"], r))
    for k, ref in (("dA", g["dA"]), ("dD", g["dD"]), ("ddt_bias", g["ddt_bias"])):
        e = rel_err(to_np(o1[k]), ref)
        assert e <= TOL[(io, "bwd")], (k, e)
    _, rdw, rdb = oracle.conv_bwd(x, p["w"], p["bias"], pr, to_np(o1["du"]))
    assert rel_err(to_np(o1["dw"]), rdw) <= TOL[(io, "bwd")]
    assert rel_err(to_np(o1["db"]), rdb) <= TOL[(io, "bwd")]


def test_programmatic_launch_overlap_is_bit_identical(monkeypatch):
    """pm_selective_scan_fwd_bwd launches the scan bwd programmatically behind
    its own scan fwd (it starts on the SMs the fwd's last CTAs leave and
    waits per segment on the fwd's release counts).  It must give exactly
    the results of separate fwd and bwd calls (plain launches), on the
    bench's 1.4B launch, over repeated back-to-back pairs (schedule counters
    self-reset between bwd launches)."""
    cfg = workload.CONFIGS["1.4b"]
    pos_np, valid, T, P = build(cfg, cfg.R)
    pos = torch.as_tensor(pos_np, device="cuda")
    u = pm.pm_causal_conv1d_fwd(T["x"], P["w"], P["bias"], pos)
    R, Dn, L = u.shape
    st = torch.empty(pm.pm_selective_scan_state_bytes(R, Dn, L, cfg.N) // 4,
                     dtype=torch.float32, device="cuda")
    y = torch.empty_like(u)
    ws = torch.empty(pm.pm_selective_scan_bwd_workspace(R, Dn, L, cfg.N), dtype=torch.uint8,
                     device="cuda")
    out = dict(du=torch.empty_like(u), ddt=torch.empty_like(u))
    args = (u, T["dt"], P["A"], T["B"], T["C"], P["D"], P["dt_bias"], pos)

    pm.pm_selective_scan_fwd(*args, y=y, states=st)
    ref = {k: v.clone() for k, v in pm.pm_selective_scan_bwd(
        *args, T["dy"], states=st, out=out, workspace=ws).items()}
    y_ref = y.clone()
    torch.cuda.synchronize()
    monkeypatch.setenv("PM_PDL", "1")  # programmatic whatever the load heuristic says
    for _ in range(4):
        y.zero_()
        _, got = pm.pm_selective_scan_fwd_bwd(*args, T["dy"], st, out=y, grads=out, workspace=ws)
        torch.cuda.synchronize()
        assert torch.equal(y, y_ref)
        for k in ref:
            assert torch.equal(got[k], ref[k]), k


def test_fwd_bwd_rejects_overlapping_buffers():
    """The fused call lets the bwd start before the fwd ends, so a bwd output
    overlapping a fwd output or an input is an argument error (pm.h)."""
    cfg = workload.Shape("ov", 1, 256, 64, 16, 4, "f32")
    rows = [[100, 156]]
    pos_np, valid = workload.pos_from_rows(rows, cfg.L)
    T = workload.row_tensors(torch, cfg, [0], valid, device="cuda")
    P = workload.params(torch, cfg, device="cuda")
    pos = torch.as_tensor(pos_np, device="cuda")
    st = torch.empty(pm.pm_selective_scan_state_bytes(1, cfg.Dn, cfg.L, cfg.N) // 4,
                     dtype=torch.float32, device="cuda")
    args = (T["x"], T["dt"], P["A"], T["B"], T["C"], P["D"], P["dt_bias"], pos)
    y = torch.empty_like(T["x"])
    with pytest.raises(pm.PMError) as e:  # du aliases the forward output y
        pm.pm_selective_scan_fwd_bwd(*args, T["dy"], st, out=y, grads=dict(du=y))
    assert e.value.name == "PM_ERR_INVALID_ARG"
    with pytest.raises(pm.PMError) as e:  # ddt aliases the input dt
        pm.pm_selective_scan_fwd_bwd(*args, T["dy"], st, out=y, grads=dict(ddt=T["dt"]))
    assert e.value.name == "PM_ERR_INVALID_ARG"
    _, g = pm.pm_selective_scan_fwd_bwd(*args, T["dy"], st, out=y)
    torch.cuda.synchronize()
    g2 = pm.pm_selective_scan_bwd(*args, T["dy"], states=st)
    torch.cuda.synchronize()
    for k in ("du", "ddt", "dA", "dB", "dC", "dD", "ddt_bias"):
        assert torch.equal(g[k], g2[k]), k
