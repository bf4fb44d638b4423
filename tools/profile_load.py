"""K0 under a profiler: RMAT generated on the device, its edge arrays exported
to device tensors, then ONE lmx_load_graph from them (the profiled region,
between cudaProfilerStart/Stop)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1302_4587_b200 import Engine  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
eng = Engine(0)
eng.set_stream(torch.cuda.current_stream().cuda_stream)
eng.gen_rmat(scale, 16, 0.57, 0.19, 0.19, seed=1, permute=True)
n, m = eng.graph_size()
du, dv, dw = eng.export_graph_device()
eng.load_graph_device(n, du, dv, dw)   # warm (allocation cache)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
eng.load_graph_device(n, du, dv, dw)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("load ms", eng.last_timing()["setup_ms"], "n", n, "m", m)
