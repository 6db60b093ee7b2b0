"""Run-to-run and launch-shape agreement of the scan fwd+bwd on a config:
full launch repeated (fused fwd_bwd, PDL as the library chooses), with
PM_NO_PDL=1, and a single-row launch of the last row; prints per-tensor
mismatch counts and max |diff|."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import oracle, workload
import paper_2408_03865_b200 as pm

name = sys.argv[1] if len(sys.argv) > 1 else "2.8b"
cfg = workload.CONFIGS[name]
R = cfg.R
n = int(R * cfg.L / 500) + 64
lens = workload.lengths_stream(cfg.name, n)
row, off, nr = oracle.plan_fifo(lens, cfg.L)
keep = row < R
rows = workload.rows_from_plan(lens[keep], row[keep], off[keep], R)
pos_np, valid = workload.pos_from_rows(rows, cfg.L)
T = workload.row_tensors(torch, cfg, list(range(R)), valid, device="cuda")
P = workload.params(torch, cfg, device="cuda")
pos = torch.as_tensor(pos_np, device="cuda")

def run(pos, T, fused=True, poison=False):
    u = pm.pm_causal_conv1d_fwd(T["x"], P["w"], P["bias"], pos)
    Rr, Dn, L = u.shape
    st = torch.empty(pm.pm_selective_scan_state_bytes(Rr, Dn, L, cfg.N) // 4, dtype=torch.float32, device="cuda")
    ws = torch.empty(pm.pm_selective_scan_bwd_workspace(Rr, Dn, L, cfg.N), dtype=torch.uint8, device="cuda")
    y = torch.empty_like(u)
    outs = dict(du=torch.empty_like(u), ddt=torch.empty_like(u))
    if poison:  # NaN everywhere the library may not read before writing
        st.fill_(float("nan")); ws.view(torch.float32)[: ws.numel() // 4].fill_(float("nan"))
        y.fill_(float("nan"));
        for v in outs.values(): v.fill_(float("nan"))
    args = (u, T["dt"], P["A"], T["B"], T["C"], P["D"], P["dt_bias"], pos)
    if fused:
        y, g = pm.pm_selective_scan_fwd_bwd(*args, T["dy"], st, out=y, grads=outs, workspace=ws)
    else:
        y, _ = pm.pm_selective_scan_fwd(*args, states=st)
        g = pm.pm_selective_scan_bwd(*args, T["dy"], states=st)
    torch.cuda.synchronize()
    return dict(y=y, **{k: v for k, v in g.items() if v is not None})

def cmp(tag, a, b, r=None):
    out = []
    for k in ("y", "du", "ddt", "dB", "dC", "dA", "dD", "ddt_bias"):
        x, y = a[k], b[k]
        if r is not None and k not in ("dA", "dD", "ddt_bias"):
            x = x[r:r + 1]
        if x.shape != y.shape:
            continue
        d = (x.float() - y.float()).abs()
        out.append(f"{k}:{int((d > 0).sum())}/{d.numel()} max {float(d.max()):.3g}")
    print(tag, " ".join(out), flush=True)

ref = run(pos, T)
for i in range(3):
    cmp(f"poisoned {i}", run(pos, T, poison=True), ref)
for i in range(3):
    cmp(f"fused rerun {i}", run(pos, T), ref)
os.environ["PM_NO_PDL"] = "1"
cmp("no-pdl fused", run(pos, T), ref)
cmp("separate", run(pos, T, fused=False), ref)
del os.environ["PM_NO_PDL"]
os.environ["PM_FWD_SPLIT"] = "1"
r = R - 1
T1 = {k: v[r:r + 1].contiguous() for k, v in T.items()}
one = run(pos[r:r + 1].contiguous(), T1)
cmp("single row vs full row", ref, one, r=r)
