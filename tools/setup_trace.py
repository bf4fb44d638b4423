"""Trace K0 stages (LMX_TRACE_SETUP=1) for the device RMAT build and a pinned-host load."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1302_4587_b200 import Engine, Graph  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
eng = Engine(0)
t = time.perf_counter()
eng.gen_rmat(scale, 16, 0.57, 0.19, 0.19, seed=1, permute=True)
print("gen_rmat total ms", (time.perf_counter() - t) * 1e3, file=sys.stderr)
g = eng.export_graph()
n, m = eng.graph_size()
pu = torch.empty(m, dtype=torch.int64, pin_memory=True)
pv = torch.empty(m, dtype=torch.int64, pin_memory=True)
pw = torch.empty(m, dtype=torch.float64, pin_memory=True)
pu.numpy()[:] = g.edge_u
pv.numpy()[:] = g.edge_v
pw.numpy()[:] = g.edge_weight
del g
for _ in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    du, dv, dw = pu.cuda(non_blocking=True), pv.cuda(non_blocking=True), pw.cuda(non_blocking=True)
    torch.cuda.synchronize()
    print("plain torch H2D ms", (time.perf_counter() - t) * 1e3, file=sys.stderr)
    del du, dv, dw
torch.cuda.empty_cache()
hg = Graph(n, pu.numpy(), pv.numpy(), pw.numpy())
for _ in range(4):
    t = time.perf_counter()
    eng.load_graph(hg)
    print("load_graph total ms", (time.perf_counter() - t) * 1e3, file=sys.stderr)
