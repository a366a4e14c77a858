#!/usr/bin/env python3
"""Summarise ncu captures into profiles/ (markdown + JSON).

  python tools/ncu_summary.py full  <report.ncu-rep> <out.md> [--traffic-json profiles/ncu_traffic.json --edge-frames N]
  python tools/ncu_summary.py launches <launches.csv> <out.md>

`full` lists, per profiled kernel: duration, DRAM bytes read/written, DRAM
throughput, issue-slot use, occupancy, registers and the top stall reasons.
`launches` aggregates a `--metrics gpu__time_duration.sum` launch list into
per-kernel totals and shares (cold-cache, serialised: compare shares only).
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict


def _csv(args):
    out = subprocess.run(["ncu", *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def full(rep, out_md, traffic_json=None, edge_frames=None):
    rows = _csv(["-i", rep, "--page", "raw"])
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and
                  h.endswith("_per_issue_active.ratio")]
    lines = ["| # | kernel | grid | dur (us) | DRAM read (MB) | DRAM write (MB) | DRAM GB/s | DRAM % peak | issue busy % |"
             " occupancy % | regs | top stalls (warps per issue) |", "|" + "---|" * 12]
    res = []
    for r in rows[2:]:
        def g(k, default=""):
            return r[ix[k]] if k in ix else default
        name = g("Kernel Name")
        dur = float(g("gpu__time_duration.sum", "0") or 0)
        rd = float(g("dram__bytes_read.sum", "0") or 0)
        wr = float(g("dram__bytes_write.sum", "0") or 0)
        def to_mb(col, v):
            unit = rows[1][ix[col]] if col in ix else ""
            return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
        rd_mb, wr_mb = to_mb("dram__bytes_read.sum", rd), to_mb("dram__bytes_write.sum", wr)
        dur_unit = rows[1][ix["gpu__time_duration.sum"]]
        dur_us = dur * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(dur_unit, 1.0)
        gbs = (rd_mb + wr_mb) * 1e6 / (dur_us * 1e-6) / 1e9 if dur_us else 0
        stalls = sorted(((float(r[ix[h]] or 0), h.replace("smsp__average_warps_issue_stalled_", "")
                          .replace("_per_issue_active.ratio", "")) for h in stall_cols), reverse=True)[:3]
        lines.append(f"| {g('ID')} | `{name[:60]}` | {g('launch__grid_size')} | {dur_us:.1f} | {rd_mb:.1f} | {wr_mb:.1f} |"
                     f" {gbs:.0f} | {g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed') or g('dram__throughput.avg.pct_of_peak_sustained_elapsed')} |"
                     f" {g('sm__inst_issued.avg.pct_of_peak_sustained_active')} |"
                     f" {g('sm__warps_active.avg.pct_of_peak_sustained_active')} | {g('launch__registers_per_thread')} |"
                     f" {', '.join(f'{b} {a:.1f}' for a, b in stalls)} |")
        res.append({"kernel": name, "grid": g("launch__grid_size"), "duration_us": dur_us, "dram_read_mb": rd_mb,
                    "dram_write_mb": wr_mb, "dram_gbs": gbs,
                    "inst_executed": float(g("smsp__inst_executed.sum", "0") or 0)})
    with open(out_md, "w") as f:
        f.write(f"ncu --set full capture `{rep}`\n\n" + "\n".join(lines) + "\n")
    if traffic_json:
        with open(traffic_json, "w") as f:
            json.dump({"source": rep, "kernels": res, "k_cn_edge_frames": edge_frames}, f, indent=1)
    print("\n".join(lines))


def launches(csv_path, out_md):
    rows = list(csv.reader(open(csv_path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {h: i for i, h in enumerate(hdr)}
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[start + 1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0]
        unit = r[ix["Metric Unit"]]
        v = float(r[ix["Metric Value"]].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
        tot[name] += v
        cnt[name] += 1
    all_t = sum(tot.values())
    lines = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k in sorted(tot, key=tot.get, reverse=True):
        lines.append(f"| `{k[:70]}` | {cnt[k]} | {tot[k]:.0f} | {100 * tot[k] / all_t:.1f} % |")
    with open(out_md, "w") as f:
        f.write(f"ncu launch list `{csv_path}` (gpu__time_duration.sum, --clock-control none; cold-cache and "
                f"serialised, compare shares only)\n\n" + "\n".join(lines) + "\n")
    print("\n".join(lines[:20]))


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "full":
        tj = sys.argv[sys.argv.index("--traffic-json") + 1] if "--traffic-json" in sys.argv else None
        ef = float(sys.argv[sys.argv.index("--edge-frames") + 1]) if "--edge-frames" in sys.argv else None
        full(sys.argv[2], sys.argv[3], tj, ef)
    else:
        launches(sys.argv[2], sys.argv[3])
