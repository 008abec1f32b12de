#!/usr/bin/env python3
"""Extract the roofline-relevant metrics of one kernel from an ncu report.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--alg-bytes B] [--out profiles/x.json]

Writes duration, DRAM bytes read/written (the `traffic` figure of bench.py's
roofline), DRAM throughput % of ncu's peak, occupancy and register counts.
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_ncu_peak",
    "dram__bytes.sum.per_second": "dram_rate",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__occupancy_limit_registers": "blocks_limit_registers",
    "launch__occupancy_limit_shared_mem": "blocks_limit_smem",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "launch__shared_mem_per_block_dynamic": "dyn_smem",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
         "byte/second": 1, "Kbyte/second": 1e3, "Mbyte/second": 1e6, "Gbyte/s": 1e9,
         "Gbyte/second": 1e9, "Tbyte/s": 1e12, "Tbyte/second": 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--alg-bytes", type=float, default=None)
    ap.add_argument("--out")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"report": a.report, "kernel": vals[hdr.index("Kernel Name")][:160]}
    for i, h in enumerate(hdr):
        if h in KEYS:
            v = vals[i].replace(",", "")
            try:
                f = float(v) * SCALE.get(units[i], 1.0)
            except ValueError:
                f = v
            out[KEYS[h]] = f
    if "dram_read" in out and "dram_write" in out:
        out["dram_bytes_per_launch"] = out["dram_read"] + out["dram_write"]
        if out.get("duration"):
            out["dram_gbs"] = out["dram_bytes_per_launch"] / out["duration"] / 1e9
    if a.alg_bytes:
        out["algorithmic_bytes"] = a.alg_bytes
        out["traffic_over_algorithmic"] = out["dram_bytes_per_launch"] / a.alg_bytes
    s = json.dumps(out, indent=1)
    if a.out:
        open(a.out, "w").write(s + "\n")
    print(s)


if __name__ == "__main__":
    main()
