"""Stage times of the C4 coarsening pipeline (per level: ratings, load, match,
contract), synchronised wall clock.  usage: python tools/coarsen_profile.py [side]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1302_4587_b200 import Engine  # noqa: E402
from paper_1302_4587_b200 import coarsen as C  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
eng = Engine(0)
eng.set_stream(torch.cuda.current_stream().cuda_stream)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    levels, final, ms = C.coarsen_mesh(side, 0, engine=eng, profile=True)
    torch.cuda.synchronize()
    print(f"rep {rep}: {len(levels)} levels -> {final}, total {(time.perf_counter() - t0) * 1e3:.1f} ms "
          f"(coarsen_mesh {ms:.1f} ms)")
for i, lv in enumerate(levels):
    print(f"  level {i:2d} n={lv.n:9d} m={lv.m:9d} matched={lv.matched:8d} rounds={len(lv.rounds):2d} "
          + " ".join(f"{k}={v:.2f}" for k, v in lv.stage_ms.items()))
