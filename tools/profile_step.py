"""One warm-up matching, then one profiled matching (cudaProfilerStart/Stop
brackets it for `ncu --profile-from-start off`)."""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1302_4587_b200 import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--steps", type=int, default=1)
args = ap.parse_args()
torch.cuda.set_device(0)
eng = Engine(0)
eng.set_stream(torch.cuda.current_stream().cuda_stream)
eng.gen_rmat(args.scale, 16, 0.57, 0.19, 0.19, seed=1, permute=True)
n, m = eng.graph_size()
mate = torch.empty(n, dtype=torch.int64, device="cuda")
ids = torch.empty(n // 2 + 1, dtype=torch.int64, device="cuda")
eng.match_device(1, mate, ids)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(args.steps):
    eng.match_device(1, mate, ids)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
rounds = eng.last_rounds()
print("scale", args.scale, "n", n, "m", m, "rounds", len(rounds), eng.last_timing())
for i, r in enumerate(rounds):
    print(i, r.edges_before, r.edges_matched, r.edges_removed)
