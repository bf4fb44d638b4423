"""Time the round loop of one liblmx build (LMX_LIBRARY) on an RMAT graph."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1302_4587_b200 import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--er", action="store_true", help="the er24unit family (unit weights, compacting loop)")
ap.add_argument("--compact", action="store_true", help="force the compacting loop (LMX_OPT_ALGO 0)")
ap.add_argument("--no-kt", action="store_true", help="no per-kernel timeline (persistent loops stay on)")
args = ap.parse_args()
eng = Engine(0)
if args.compact:
    eng.set_algo("compact")
if args.er:
    eng.gen_er(args.scale, 4, seed=1, unit=True)
else:
    eng.gen_rmat(args.scale, 16, 0.57, 0.19, 0.19, seed=1, permute=True)
n, m = eng.graph_size()
mate = torch.empty(n, dtype=torch.int64, device="cuda")
ids = torch.empty(n // 2 + 1, dtype=torch.int64, device="cuda")
eng.match_device(1, mate, ids)
eng.set_kernel_timing(not args.no_kt)
best = None
for _ in range(args.steps):
    eng.match_device(1, mate, ids)
    t = eng.last_timing()
    if best is None or t["rounds_ms"] < best["rounds_ms"]:
        best = t
print(os.path.basename(os.environ.get("LMX_LIBRARY", "default")),
      "rounds_ms %.3f round_k %.3f match_k %.3f hist_k %.3f out %.3f" % (
          best["rounds_ms"], best["round_kernel_ms"], best["match_kernel_ms"], best["hist_kernel_ms"],
          best["output_ms"]))
