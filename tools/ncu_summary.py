"""Summarise ncu reports into profiles/ (tracked evidence).

usage: python tools/ncu_summary.py TAG gpurun_out/TAG_scan.ncu-rep [more.ncu-rep ...]
         [--launches gpurun_out/TAG_launches.csv] [--config 1.4b]
Writes profiles/TAG_ncu_summary.md, profiles/TAG_launches.csv (copy) and
updates profiles/ncu_traffic.json (dram read+write bytes per launch per
kernel, read by bench.py for the roofline "traffic" field).
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "smsp__inst_executed.sum": "warp_instr",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_%",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_%",
    "launch__registers_per_thread": "regs",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_%",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_%",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_%",
    "sm__cycles_active.avg": "sm_cycles_active",
    "gpc__cycles_elapsed.max": "cycles_elapsed",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}


def kind(name):
    for k in ("scan_bwd_finalize_bc", "scan_bwd_finalize_param", "scan_bwd_wide_kernel", "scan_bwd_kernel", "scan_fwd",
              "conv_bwd_finalize", "conv_bwd", "conv_fwd", "pack"):
        if k in name:
            return {"scan_bwd_kernel": "scan_bwd", "scan_bwd_wide_kernel": "scan_bwd", "scan_fwd": "scan_fwd", "conv_bwd": "conv_bwd",
                    "conv_fwd": "conv_fwd"}.get(k, k)
    return name


def scale(v, unit):
    u = unit.lower()
    f = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12, "nsecond": 1e-9,
         "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1,
         "s": 1}.get(u, 1)
    return v * f


def read(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        m = {"kernel": d["Kernel Name"][:90]}
        for k, short in KEYS.items():
            if k in d:
                try:
                    m[short] = scale(float(d[k].replace(",", "")), units[h.index(k)])
                except ValueError:
                    m[short] = d[k]
        st = []
        for k in h:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(d[k]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        m["top_stalls"] = ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:5])
        out.append(m)
    return out


def main():
    tag = sys.argv[1]
    args = sys.argv[2:]
    launches = cfg = None
    reps = []
    i = 0
    while i < len(args):
        if args[i] == "--launches":
            launches = args[i + 1]; i += 2
        elif args[i] == "--config":
            cfg = args[i + 1]; i += 2
        else:
            reps.append(args[i]); i += 1
    cfg = cfg or "1.4b"
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lines = [f"# ncu summary {tag} (config {cfg})", "",
             "`ncu --set full --clock-control none` captures (one launch per kernel, cold "
             "replay); durations are serialised single-kernel times, not the bench's.", "",
             "| kernel | dur (us) | DRAM rd (MB) | DRAM wr (MB) | warp instr | issue % | warps % | "
             "regs | xu % | fma % | grid x block | top stalls (per issue) |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    tcfg = traffic.setdefault(cfg, {})
    traffic["capture"] = f"{tag} (profiles/{tag}_ncu_summary.md)"
    for rep in reps:
        for m in read(rep):
            g = m.get
            lines.append(
                f"| {m['kernel'][:60]} | {g('duration', 0) * 1e6:.1f} | {g('dram_read', 0) / 1e6:.1f} | "
                f"{g('dram_write', 0) / 1e6:.1f} | {g('warp_instr', 0):.3e} | {g('issue_active_%', 0):.1f} | "
                f"{g('warps_active_%', 0):.1f} | {g('regs', 0):.0f} | {g('xu_pipe_%', 0):.1f} | "
                f"{g('fma_pipe_%', 0):.1f} | {g('grid', 0):.0f} x {g('block', 0):.0f} | {m['top_stalls']} |")
            k = kind(m["kernel"])
            if k in ("scan_fwd", "scan_bwd", "conv_fwd", "conv_bwd"):
                tcfg[k] = g("dram_read", 0) + g("dram_write", 0)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    if launches:
        shutil.copy(launches, os.path.join(ROOT, "profiles", f"{tag}_launches.csv"))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
