#!/usr/bin/env python3
"""Live DRAM traffic of a kernel over ONE complete bench step.

Capture on the GPU box (every launch of the kernel in one step, DRAM bytes per launch):

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        --clock-control none -k regex:k_layer --csv --log-file gpurun_out/traffic.csv \\
        python tools/one_step.py --config C4 --schedule layered > gpurun_out/one_step.json

then here:

    python tools/ncu_traffic.py gpurun_out/traffic.csv gpurun_out/one_step.json \\
        --kernel k_layer --algo-bytes 16 --out profiles/ncu_traffic_live.json

The JSON records the summed DRAM bytes of all launches, the number of launches, the useful
edge-frames of the step (sum over coded slices of E_j x iterations over the frames that iterate,
from cvsr_stats) and their ratio: bytes per useful edge-frame against the algorithmic 16 (reading
R-9).  bench.py reports `roofline.traffic` = that ratio x the run's useful edge-frames per launch.
"""
import argparse
import csv
import json
from collections import defaultdict

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def parse(path, kernel):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {h: i for i, h in enumerate(hdr)}
    per = defaultdict(dict)
    names = {}
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        name = r[ix["Kernel Name"]]
        if kernel not in name:
            continue
        lid = r[ix["ID"]]
        v = float(r[ix["Metric Value"]].replace(",", "")) * SCALE.get(r[ix["Metric Unit"]], 1.0)
        per[lid][r[ix["Metric Name"]]] = v
        names[lid] = name.split("(")[0]
    return per, names


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("step_json")
    ap.add_argument("--kernel", default="k_layer")
    ap.add_argument("--algo-bytes", type=float, default=16.0)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    per, names = parse(a.csv, a.kernel)
    step = json.loads([ln for ln in open(a.step_json) if ln.startswith("{")][-1])
    rd = sum(d.get("dram__bytes_read.sum", 0.0) for d in per.values())
    wr = sum(d.get("dram__bytes_write.sum", 0.0) for d in per.values())
    tm = sum(d.get("gpu__time_duration.sum", 0.0) for d in per.values())
    by_kernel = defaultdict(lambda: [0, 0.0, 0.0])
    for lid, d in per.items():
        k = by_kernel[names[lid]]
        k[0] += 1
        k[1] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        k[2] += d.get("gpu__time_duration.sum", 0.0)
    ef = float(step["edge_frames"])
    out = {"config": step["config"], "schedule": step["schedule"], "kernel": a.kernel, "launches": len(per),
           "dram_read_bytes": rd, "dram_write_bytes": wr, "useful_edge_frames": ef,
           "bytes_per_useful_edge_frame": (rd + wr) / ef, "algorithmic_bytes_per_edge_frame": a.algo_bytes,
           "wasted_fraction": 1.0 - a.algo_bytes * ef / (rd + wr),
           "ncu_time_s": tm, "ncu_dram_gbs": (rd + wr) / tm / 1e9 if tm else None,
           "per_instantiation": {k: {"launches": v[0], "dram_bytes": v[1], "ncu_time_s": v[2]}
                                 for k, v in sorted(by_kernel.items())},
           "source": {"csv": a.csv, "step": a.step_json}}
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("launches", "bytes_per_useful_edge_frame", "wasted_fraction",
                                           "ncu_dram_gbs")}))


if __name__ == "__main__":
    main()
