"""Per-round kernel durations of one match on an RMAT graph (LMX_OPT_KERNEL_TIMING)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1302_4587_b200 import Engine  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
eng = Engine(0)
if len(sys.argv) > 2:
    eng.set_algo(sys.argv[2])
eng.gen_rmat(scale, 16, 0.57, 0.19, 0.19, seed=1, permute=True)
n, m = eng.graph_size()
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
rounds = eng.last_rounds()
print(f"n={n} m={m} layout={eng.layout()} relabeled={eng.relabeled()} algo={eng.algo()} setup_ms={eng.last_timing()['setup_ms']:.1f}")
print(" r   edges_before  matched      round_ms  match_ms  GB/s(16B/edge read)")
tr = tm = 0.0
for r, (a, b) in enumerate(best):
    eb = rounds[r].edges_before if r < len(rounds) else 0
    mt = rounds[r].edges_matched if r < len(rounds) else 0
    tr += a
    tm += b
    print(f"{r:2d} {eb:14d} {mt:9d} {a:9.3f} {b:9.3f} {16 * eb / max(a, 1e-9) / 1e6:9.0f}")
print(f"total round {tr:.3f} match {tm:.3f} sum {tr + tm:.3f}")
