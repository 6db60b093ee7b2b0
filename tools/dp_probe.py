import os, sys
sys.path.insert(0, "/root/repo")
import torch
from tests.test_gpu_dp import _cfg, _layout, _run_rows
cfg = _cfg()
layout = _layout(cfg, 8)
for ts in ["0", "1"]:
    os.environ["PM_TSPLIT"] = ts
    _, a = _run_rows(cfg, [4, 5, 6, 7], layout)
    _, b = _run_rows(cfg, list(range(8)), layout)
    for k in ("du", "ddt", "dB", "dC", "y"):
        x, y = a[k], b[k][4:8]
        d = (x.float() - y.float()).abs()
        nz = torch.nonzero(d > 0)
        print(ts, k, int((d > 0).sum()), float(d.max()), nz[:5].tolist() if len(nz) else "")
