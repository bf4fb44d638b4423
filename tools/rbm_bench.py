"""RBM vs local max on device-built RMAT graphs: rounds, device time, validity."""
import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1302_4587_b200 import Engine
for scale in (22, 24):
    eng = Engine(0)
    eng.gen_rmat(scale, 16, 0.57, 0.19, 0.19, seed=1, permute=True)
    g = eng.export_graph()
    for _ in range(2):
        t = time.perf_counter(); m, tr = eng.rbm(g, 1); dt = time.perf_counter() - t
    chk, wgt = eng.validate(m)
    mm, tr2 = eng.match(g, 1, True)
    print(f"rmat{scale}: rbm rounds {len(tr.rounds)} device {tr.device_millis:.1f} ms wall {dt*1e3:.0f} ms matched {len(m.sorted_edge_ids())} valid {chk.valid} maximal {chk.maximal}; localmax rounds {len(tr2.rounds)} {tr2.device_millis:.1f} ms", flush=True)
    eng.close()
