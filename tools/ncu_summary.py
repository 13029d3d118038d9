"""Summarise ncu outputs for profiles/: launch-list shares and the key
metrics of a --set full capture (run here, on the CPU box)."""
import csv
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = defaultdict(lambda: [0, 0.0])
    for r in rows[h + 1:]:
        if len(r) > vi:
            name = r[ki].split("(")[0][:90]
            tot[name][0] += 1
            tot[name][1] += float(r[vi].replace(",", ""))
    allns = sum(v[1] for v in tot.values())
    return [{"kernel": k, "launches": v[0], "total_us": round(v[1] / 1e3, 1), "avg_us": round(v[1] / v[0] / 1e3, 2),
             "share": round(v[1] / allns, 4)} for k, v in sorted(tot.items(), key=lambda kv: -kv[1][1])]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for k in KEYS:
            if k in hdr:
                d[k] = f"{r[hdr.index(k)]} {units[hdr.index(k)]}".strip()
        res.append(d)
    return res


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launches(path) if kind == "launches" else full(path), indent=1))
