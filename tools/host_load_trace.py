"""Load from page-locked host arrays (bench.py's e2e leg) under several host
thread counts, with LMX_TRACE_SETUP stage times; plus the raw host numbers
(torch H2D of the int64 arrays, numpy narrowing).  usage: host_load_trace.py [scale]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if not os.environ.get("TRACE_OFF"):
    os.environ["LMX_TRACE_SETUP"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1302_4587_b200 import Engine, Graph  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
eng = Engine(0)
if os.environ.get("TRACE_TORCH_STREAM"):
    eng.set_stream(torch.cuda.current_stream().cuda_stream)   # as bench.py does
eng.gen_rmat(scale, 16, 0.57, 0.19, 0.19, seed=1, permute=True)
g0 = eng.export_graph()
n, m = g0.num_vertices, len(g0.edge_u)
pu = torch.empty(m, dtype=torch.int64, pin_memory=True)
pv = torch.empty(m, dtype=torch.int64, pin_memory=True)
pw = torch.empty(m, dtype=torch.float64, pin_memory=True)
pu.numpy()[:] = g0.edge_u
pv.numpy()[:] = g0.edge_v
pw.numpy()[:] = g0.edge_weight
g = Graph(n, pu.numpy(), pv.numpy(), pw.numpy())
out = np.empty(m, dtype=np.uint32)
t = time.perf_counter()
np.copyto(out, pu.numpy(), casting="unsafe")
print(f"numpy narrow (1 thread) {m * 12 / (time.perf_counter() - t) / 1e9:.1f} GB/s", file=sys.stderr)
d = torch.empty(m, dtype=torch.int64, device="cuda")
for _ in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    d.copy_(pu, non_blocking=True)
    torch.cuda.synchronize()
    print(f"torch H2D int64 {m * 8 / (time.perf_counter() - t) / 1e9:.1f} GB/s", file=sys.stderr)
del d
configs = [(os.cpu_count(), 4, 1 << 19, 1), (0, 0, 0, 0)]
if len(sys.argv) > 2:
    configs = [tuple(int(x) for x in c.split(",")) for c in sys.argv[2:]]
for th, ring, block, nt in configs:
    for k in ("LMX_LOAD_THREADS", "LMX_LOAD_RING", "LMX_LOAD_LEGACY", "LMX_LOAD_BLOCK", "LMX_LOAD_NT"):
        os.environ.pop(k, None)
    if th:
        os.environ["LMX_LOAD_THREADS"] = str(th)
        os.environ["LMX_LOAD_RING"] = str(ring)
        os.environ["LMX_LOAD_BLOCK"] = str(block)
        os.environ["LMX_LOAD_NT"] = str(nt)
    else:
        os.environ["LMX_LOAD_LEGACY"] = "1"
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        print(f"--- threads {th or 'legacy'} ring {ring} block {block} nt {nt} rep {rep}", file=sys.stderr, flush=True)
        eng.load_graph(g)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        eng.match_raw(1, True)
        t2 = time.perf_counter()
        print(f"load_graph total ms {(t1 - t) * 1e3:.1f}; + match_raw (D2H) ms {(t2 - t1) * 1e3:.1f}",
              file=sys.stderr, flush=True)
