"""GPU tests of the binding's argument checks and of pointer-alignment
fallbacks (the C ABI receives void pointers only, so the binding checks
dtype and shape; the library picks the vector/TMA path only for 16-byte
aligned pointers)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2408_03865_b200 as pm
import workload

pytestmark = pytest.mark.gpu


def _problem(io="f32", R=2, L=256, Dn=64, N=16):
    cfg = workload.Shape("api", R, L, Dn, N, 4, io)
    rows = [[100, 56, 100], [7, 200]][:R]
    pos_np, valid = workload.pos_from_rows(rows, L)
    T = workload.row_tensors(torch, cfg, list(range(R)), valid, device="cuda")
    P = workload.params(torch, cfg, device="cuda")
    return torch.as_tensor(pos_np, device="cuda"), T, P


def test_binding_rejects_wrong_dtypes_and_shapes():
    pos, T, P = _problem()
    args = lambda **kw: {**dict(u=T["x"], dt=T["dt"], A=P["A"], B=T["B"], C=T["C"],
                                Dskip=P["D"], dt_bias=P["dt_bias"], pos=pos), **kw}
    with pytest.raises(TypeError, match="pos"):  # torch.arange-style int64 positions
        pm.pm_selective_scan_fwd(**args(pos=pos.long()))
    with pytest.raises(TypeError, match="B"):  # fp32 B next to bf16 u
        pm.pm_selective_scan_fwd(**args(u=T["x"].bfloat16(), dt=T["dt"].bfloat16(),
                                        C=T["C"].bfloat16()))
    with pytest.raises(ValueError, match="B"):  # B with another N
        pm.pm_selective_scan_fwd(**args(B=T["B"][:, :8].contiguous()))
    with pytest.raises(ValueError, match="dt"):  # dt with another L
        pm.pm_selective_scan_fwd(**args(dt=T["dt"][..., :128].contiguous()))
    with pytest.raises(TypeError, match="A"):
        pm.pm_selective_scan_fwd(**args(A=P["A"].double()))
    y, st = pm.pm_selective_scan_fwd(**args())
    with pytest.raises(TypeError, match="dy"):
        pm.pm_selective_scan_bwd(**args(), dy=T["dy"].bfloat16(), states=st)
    with pytest.raises(ValueError, match="dB"):
        pm.pm_selective_scan_bwd(**args(), dy=T["dy"], states=st,
                                 out=dict(dB=torch.empty(1, 16, 256, device="cuda")))
    with pytest.raises(TypeError, match="pos"):
        pm.pm_causal_conv1d_fwd(T["x"], P["w"], P["bias"], pos.long())
    with pytest.raises(ValueError, match="bias"):
        pm.pm_causal_conv1d_fwd(T["x"], P["w"], P["bias"][:10].contiguous(), pos)


@pytest.mark.parametrize("io", ["f32", "bf16"])
def test_pos_4byte_aligned_view(io):
    """pos that is 4- but not 16-byte aligned (a view at offset 1): the scan
    bwd must not take the TMA / 16-byte cp.async path for it (that would be a
    misaligned-address fault) and must give the aligned run's results."""
    pos, T, P = _problem(io)
    R, L = pos.shape
    T = {k: v.to(torch.bfloat16 if io == "bf16" else torch.float32) for k, v in T.items()}
    buf = torch.empty(R * L + 1, dtype=torch.int32, device="cuda")
    pos_off = buf[1:].view(R, L)
    pos_off.copy_(pos)
    assert pos_off.data_ptr() % 16 != 0 and pos_off.data_ptr() % 4 == 0
    out = {}
    for name, p in (("aligned", pos), ("offset", pos_off)):
        u = pm.pm_causal_conv1d_fwd(T["x"], P["w"], P["bias"], p)
        y, st = pm.pm_selective_scan_fwd(u, T["dt"], P["A"], T["B"], T["C"], P["D"],
                                         P["dt_bias"], p)
        g = pm.pm_selective_scan_bwd(u, T["dt"], P["A"], T["B"], T["C"], P["D"], P["dt_bias"], p,
                                     T["dy"], states=st)
        dx, dw, db = pm.pm_causal_conv1d_bwd(T["x"], P["w"], P["bias"], p, g["du"])
        torch.cuda.synchronize()
        out[name] = dict(u=u, y=y, dx=dx, dw=dw, db=db, **g)
    for k, v in out["aligned"].items():
        # the unaligned launch may take the scalar path (another summation
        # order of nothing: every per-lane recurrence is the same sequence of
        # operations), so per-token outputs agree to rounding of the
        # cross-channel dB/dC partials only
        tol = 2e-2 if v.dtype == torch.bfloat16 else 1e-5
        torch.testing.assert_close(out["offset"][k], v, rtol=tol, atol=tol, msg=k)
