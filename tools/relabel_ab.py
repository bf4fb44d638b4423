"""A/B: degree-descending relabelling on / off for one workload: device load
time (K0) and per-matching time.  usage: relabel_ab.py [scale]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1302_4587_b200 import Engine  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
eng = Engine(0)
eng.set_stream(torch.cuda.current_stream().cuda_stream)
eng.gen_rmat(scale, 16, 0.57, 0.19, 0.19, seed=1, permute=True)
n, m = eng.graph_size()
du, dv, dw = eng.export_graph_device()
ref = None
for mode in ("on", "off", "on", "off"):
    eng.set_relabel(mode)
    loads = []
    for _ in range(2):
        eng.load_graph_device(n, du, dv, dw)
        loads.append(eng.last_timing()["setup_ms"])
    ts = []
    for _ in range(6):
        mate, ids, rounds = eng.match_raw(1, True)
        ts.append(eng.last_timing()["rounds_ms"])
    if ref is None:
        ref = (mate.copy(), ids.copy())
    assert np.array_equal(mate, ref[0]) and np.array_equal(ids, ref[1])
    print(f"relabel {mode}: relabeled={eng.relabeled()} load ms {min(loads):.1f}  match rounds_ms "
          f"min {min(ts[1:]):.3f} median {sorted(ts[1:])[2]:.3f}", flush=True)
