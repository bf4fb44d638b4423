"""Per-round, per-phase warp-cycle shares of the round kernel (LMX_PHASE_TIMING build)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1302_4587_b200 import Engine  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
eng = Engine(0)
eng.gen_rmat(scale, 16, 0.57, 0.19, 0.19, seed=1, permute=True)
n, m = eng.graph_size()
mate = torch.empty(n, dtype=torch.int64, device="cuda")
ids = torch.empty(n // 2 + 1, dtype=torch.int64, device="cuda")
eng.match_device(1, mate, ids)
buf = np.zeros(64 * 5, dtype=np.uint64)
eng._lib.lmx_debug_phase_cycles(ctypes.c_void_p(buf.ctypes.data), 1)
eng.set_kernel_timing(True)
eng.match_device(1, mate, ids)
eng._lib.lmx_debug_phase_cycles(ctypes.c_void_p(buf.ctypes.data), 1)
print(eng.last_timing())
c = buf.reshape(64, 5)[:, :4].astype(np.float64)
names = ["hubs(b3,b4)", "warp(b2)", "grp8(b1)", "thread(b0)"]
for r in range(16):
    if c[r].sum() == 0:
        continue
    print(r, " ".join(f"{nm}={100 * x / c[r].sum():5.1f}%" for nm, x in zip(names, c[r])), f"warp-Gcyc={c[r].sum() / 1e9:.2f}")
