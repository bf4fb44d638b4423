"""K0 stage times (LMX_TRACE_SETUP=1) of lmx_load_graph from DEVICE-resident
edge arrays (bench.py's load_device_ms).  usage: python tools/load_trace.py [scale] [rmat|er]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1302_4587_b200 import Engine  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
family = sys.argv[2] if len(sys.argv) > 2 else "rmat"
eng = Engine(0)
eng.set_stream(torch.cuda.current_stream().cuda_stream)
if family == "er":   # same m, no hubs (random weights via a U[0,1) fill of the unit graph's weights)
    eng.gen_er(scale, 16, seed=1, unit=False)
else:
    eng.gen_rmat(scale, 16, 0.57, 0.19, 0.19, seed=1, permute=True)
n, m = eng.graph_size()
du, dv, dw = eng.export_graph_device()
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    print(f"--- load {rep}", file=sys.stderr, flush=True)
    eng.load_graph_device(n, du, dv, dw)
    torch.cuda.synchronize()
    print(f"load_graph_device total ms {(time.perf_counter() - t) * 1e3:.1f} (events {eng.last_timing()['setup_ms']:.1f})",
          file=sys.stderr, flush=True)
