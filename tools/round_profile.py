"""Per-round kernel durations and device counters of one match on an RMAT graph.

usage: python tools/round_profile.py [scale] [auto|compact|scan] [rmat|er]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1302_4587_b200 import Engine  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
eng = Engine(0)
if len(sys.argv) > 2:
    eng.set_algo(sys.argv[2])
if len(sys.argv) > 3 and sys.argv[3] == "er":
    eng.gen_er(scale, 4, seed=1, unit=True)
else:
    eng.gen_rmat(scale, 16, 0.57, 0.19, 0.19, seed=1, permute=True)
n, m = eng.graph_size()
setup_ms = eng.last_timing()["setup_ms"]
mate = torch.empty(n, dtype=torch.int64, device="cuda")
ids = torch.empty(n // 2 + 1, dtype=torch.int64, device="cuda")
for _ in range(2):
    eng.match_device(1, mate, ids)
eng.set_kernel_timing(True)
best = None
for _ in range(3):
    eng.match_device(1, mate, ids)
    kt = eng.last_kernel_times()
    if best is None or sum(a + b for a, b in kt) < sum(a + b for a, b in best):
        best = kt
        ctr = eng.last_round_counters()
rounds = eng.last_rounds()
algo = eng.algo()
print(f"n={n} m={m} layout={eng.layout()} relabeled={eng.relabeled()} algo={algo} setup_ms={setup_ms:.1f}")
cols = "|A_r|  |M|b0  |M|b1  |M|b2  |M|b3+" if algo == "scan" else "b0 b1 b2 b3 b4"
print(f" r   edges_before  matched  round_ms match_ms   slot_reads  {cols}")
tr = tm = 0.0
for r, (a, b) in enumerate(best):
    eb = rounds[r].edges_before if r < len(rounds) else 0
    mt = rounds[r].edges_matched if r < len(rounds) else 0
    tr += a
    tm += b
    c = ctr[r] if r < len(ctr) else [0] * 8
    print(f"{r:2d} {eb:14d} {mt:8d} {a:9.3f} {b:8.3f} {c[0]:12d}  " + " ".join(f"{int(x):9d}" for x in c[3:8]))
print(f"total round {tr:.3f} match {tm:.3f} sum {tr + tm:.3f}")
