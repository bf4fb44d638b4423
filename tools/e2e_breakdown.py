"""Where the end-to-end step goes: load (H2D + build) vs match vs host outputs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1302_4587_b200 import Engine, Graph  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
eng = Engine(0)
eng.gen_rmat(scale, 16, 0.57, 0.19, 0.19, seed=1, permute=True)
g0 = eng.export_graph()
n, m = eng.graph_size()
pu = torch.empty(m, dtype=torch.int64, pin_memory=True)
pv = torch.empty(m, dtype=torch.int64, pin_memory=True)
pw = torch.empty(m, dtype=torch.float64, pin_memory=True)
pu.numpy()[:] = g0.edge_u
pv.numpy()[:] = g0.edge_v
pw.numpy()[:] = g0.edge_weight
del g0
hg = Graph(n, pu.numpy(), pv.numpy(), pw.numpy())
relabel = os.environ.get("E2E_RELABEL", "once")
for it in range(3):
    t0 = time.perf_counter()
    eng.set_relabel(relabel)
    eng.load_graph(hg)
    t1 = time.perf_counter()
    mate, ids, rounds = eng.match_raw(1, True)
    t2 = time.perf_counter()
    tm = eng.last_timing()
    print(f"load {1e3 * (t1 - t0):.1f} ms (device setup {tm['setup_ms']:.1f})  match_raw {1e3 * (t2 - t1):.1f} ms "
          f"(rounds {tm['rounds_ms']:.1f} + outputs {tm['output_ms']:.1f})", flush=True)
