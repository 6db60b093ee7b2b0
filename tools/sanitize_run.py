"""One step of the hot path (conv fwd, fused scan fwd+bwd, conv bwd, plus the
separate fwd/bwd calls and the recompute path) for compute-sanitizer runs.
usage: python tools/sanitize_run.py CONFIG   (tiny | small | 130m | a workload.CONFIGS name)
PM_PDL=1 forces the programmatic bwd launch behind the fwd."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import oracle  # noqa: E402  (planner only: the layout of the rows)
import paper_2408_03865_b200 as pm  # noqa: E402
import workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
if name == "small":
    cfg = workload.Shape("small", 2, 2048, 256, 16, 4, "bf16")
else:
    cfg = workload.CONFIGS[name]
if cfg.layout == "explicit":
    rows = cfg.rows
else:
    lens = workload.lengths_stream(cfg.name, cfg.R * cfg.L // 200 + 64)
    row, off, nr = oracle.plan_fifo(lens, cfg.L)
    keep = row < cfg.R
    rows = workload.rows_from_plan(lens[keep], row[keep], off[keep], cfg.R)
pos_np, valid = workload.pos_from_rows(rows, cfg.L)
pos = torch.as_tensor(pos_np, device="cuda")
T = workload.row_tensors(torch, cfg, list(range(cfg.R)), valid, device="cuda")
P = workload.params(torch, cfg, device="cuda")
R, Dn, L, N = cfg.R, cfg.Dn, cfg.L, cfg.N
u = pm.pm_causal_conv1d_fwd(T["x"], P["w"], P["bias"], pos)
st = torch.empty(pm.pm_selective_scan_state_bytes(R, Dn, L, N) // 4, dtype=torch.float32,
                 device="cuda")
args = (u, T["dt"], P["A"], T["B"], T["C"], P["D"], P["dt_bias"], pos)
y, g = pm.pm_selective_scan_fwd_bwd(*args, T["dy"], st, out=torch.empty_like(u))
dx, dw, db = pm.pm_causal_conv1d_bwd(T["x"], P["w"], P["bias"], pos, g["du"])
y2, _ = pm.pm_selective_scan_fwd(*args, states=st)
g2 = pm.pm_selective_scan_bwd(*args, T["dy"], states=st)
g3 = pm.pm_selective_scan_bwd(*args, T["dy"], states=None)  # recompute path (own fwd + PDL)
torch.cuda.synchronize()
for k in ("du", "ddt", "dA", "dB", "dC"):
    assert torch.equal(g[k], g2[k]) and torch.equal(g[k], g3[k]), k
assert torch.equal(y, y2)
print("ok", name, {k: float(v.float().abs().max()) for k, v in g.items() if v is not None})
