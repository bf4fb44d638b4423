"""Per-partition device memory of the distributed RMAT build + matching.

All p partitions run in this process on one GPU (LocalComm), so the sum must
fit one B200; each rank's own numbers are what one GPU per rank would hold.
usage: python tools/dist_memory.py scale p [p ...]  -> one JSON line per p
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1302_4587_b200 import Engine  # noqa: E402
from paper_1302_4587_b200.dist import local_max_dist_rmat  # noqa: E402

scale = int(sys.argv[1])
for p in [int(x) for x in sys.argv[2:]]:
    t0 = time.perf_counter()
    matching, trace, db = local_max_dist_rmat(p, scale, 1, True, graph_seed=1, permute=True)
    dt = time.perf_counter() - t0
    print(json.dumps({"scale": scale, "p": p, "m": trace.rounds[0].edges_before, "rounds": len(trace.rounds),
                      "matched": int(matching.size),
                      "rank_bytes_after_load_GB": [round(x[0] / 1e9, 2) for x in db],
                      "rank_peak_bytes_GB": [round(x[1] / 1e9, 2) for x in db],
                      "wall_s": round(dt, 1)}), flush=True)
if len(sys.argv) > 2 and os.environ.get("SINGLE"):
    eng = Engine(0)
    eng.peak_device_bytes(reset=True)
    eng.gen_rmat(scale, 16, seed=1, permute=True)
    print(json.dumps({"scale": scale, "p": 1, "single_gpu_bytes_after_load_GB": round(eng.device_bytes() / 1e9, 2),
                      "single_gpu_peak_GB": round(eng.peak_device_bytes() / 1e9, 2)}))
