"""Key counters of an ncu --set full capture -> profiles/<round>/<name>.metrics.json,
and (optionally) the per-launch DRAM traffic into profiles/ncu_summary.json.

usage: python tools/ncu_extract.py REPORT.ncu-rep OUT.metrics.json [summary_key]
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    key = sys.argv[3] if len(sys.argv) > 3 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    d = {h: [v, u] for h, u, v in zip(head, units, vals)}
    res = {k: d[k] for k in KEYS if k in d}
    stalls = {h.replace("smsp__average_warps_issue_stalled_", "").replace(
        "_per_issue_active.ratio", ""): float(d[h][0] or 0)
        for h in head if h.startswith("smsp__average_warps_issue_stalled_")
        and h.endswith("_per_issue_active.ratio")}
    res["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    if key:
        traffic = sum(float(d[k][0]) * SCALE.get(d[k][1], 1)
                      for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        path = os.path.join(os.path.dirname(__file__), "..", "profiles", "ncu_summary.json")
        with open(path) as f:
            summ = json.load(f)
        summ["traffic_bytes_per_launch"][key] = traffic
        summ["source"][key] = os.path.splitext(os.path.basename(out))[0].replace(".metrics", "")
        with open(path, "w") as f:
            json.dump(summ, f, indent=1)
    print(out, res.get("gpu__time_duration.sum"), res.get("dram__bytes_read.sum"))


if __name__ == "__main__":
    main()
