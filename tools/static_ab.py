"""rerandomize=False on unit weights: the static (weight, salt) layout + scan
loop against the compacting loop (both bit-identical).  Device load time
and per-matching time.  usage: static_ab.py [scale] [edge_factor]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1302_4587_b200 import Engine  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
ef = int(sys.argv[2]) if len(sys.argv) > 2 else 4
SEED = 1
eng = Engine(0)
eng.set_stream(torch.cuda.current_stream().cuda_stream)
eng.gen_er(scale, ef, seed=1, unit=True)
n, m = eng.graph_size()
du, dv, dw = eng.export_graph_device()
ref = None
for mode in ("compact", "static", "compact", "static"):
    eng.set_static_order(SEED if mode == "static" else None)
    loads = []
    for _ in range(2):
        eng.load_graph_device(n, du, dv, dw)
        loads.append(eng.last_timing()["setup_ms"])
    eng.set_static_order(None)
    ts = []
    for _ in range(8):
        mate, ids, rounds = eng.match_raw(SEED, False)
        ts.append(eng.last_timing()["rounds_ms"])
    if ref is None:
        ref = (mate.copy(), ids.copy(), list(rounds))
    assert np.array_equal(mate, ref[0]) and np.array_equal(ids, ref[1]) and list(rounds) == ref[2]
    t = sorted(ts[2:])
    print(f"er scale {scale} ef {ef} unit, rerandomize=False, {mode:7s}: algo={eng.algo()} static={eng.static_order()} "
          f"rounds={len(rounds)} load ms {min(loads):.1f}  matching ms min {t[0]:.3f} median {t[len(t) // 2]:.3f} "
          f"({m / t[len(t) // 2] / 1e6:.2f} G edges/s)", flush=True)
