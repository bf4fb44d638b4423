"""Print the key per-launch metrics of an ncu report (details page)."""
import csv
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Achieved Occupancy", "Registers Per Thread", "Compute (SM) Throughput", "Executed Ipc Active",
        "L2 Cache Throughput", "L1/TEX Cache Throughput", "Issue Slots Busy", "No Eligible",
        "Active Warps Per Scheduler", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction"]


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    idx = {n: i for i, n in enumerate(h)}
    res = {}
    for r in rows[1:]:
        name = r[idx["Metric Name"]]
        if name in WANT:
            res.setdefault(name, []).append(r[idx["Metric Value"]] + " " + r[idx["Metric Unit"]])
    return res


if __name__ == "__main__":
    for k, v in summary(sys.argv[1]).items():
        print(f"{k:38s}", " | ".join(v))
