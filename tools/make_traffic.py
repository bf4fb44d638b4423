"""profiles/traffic_<workload>.json from an ncu launch list (dram bytes per round-kernel launch)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from launches import load  # noqa: E402

csv_path, workload, out = sys.argv[1], sys.argv[2], sys.argv[3]
kernel = sys.argv[4] if len(sys.argv) > 4 else "lmx_scan_round_kernel"
K = load(csv_path)
rk = [v for v in K.values() if kernel in v["name"]]
tot_bytes = sum(v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0) for v in rk)
tot_ms = sum(v["gpu__time_duration.sum"] for v in rk)
all_ms = sum(v["gpu__time_duration.sum"] for v in K.values())
json.dump({
    "workload": workload,
    "kernel": kernel,
    "launches": len(rk),
    "bytes_per_launch": tot_bytes / max(len(rk), 1),
    "bytes_per_step": tot_bytes,
    "kernel_ms_serialised": tot_ms,
    "kernel_share_of_step": tot_ms / all_ms if all_ms else None,
    "source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
              f"--clock-control none (cold-cache, serialised launches): {os.path.basename(csv_path)}",
}, open(out, "w"), indent=1)
print(open(out).read())
