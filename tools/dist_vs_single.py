"""Diagnostic: single-GPU lmx_match vs the stepped protocol at p=1 on one RMAT graph."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
from paper_1302_4587_b200 import Engine
from paper_1302_4587_b200.dist import DistRank, TorchComm, LocalComm, run_rounds, _unpack_ids

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29555")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
st = torch.cuda.current_stream()
rm = dict(scale=scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1, permute=True)
eng = Engine(0); eng.set_stream(st.cuda_stream); eng.gen_rmat(**rm)
n, m = eng.graph_size()
mate = torch.empty(n, dtype=torch.int64, device="cuda"); ids = torch.empty(n // 2 + 1, dtype=torch.int64, device="cuda")
def single():
    return eng.match_device(1, mate, ids, True)
for _ in range(3): r = single()
torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(5): r = single()
e1.record(st); torch.cuda.synchronize()
print("single ms", e0.elapsed_time(e1) / 5, "ret", r if not hasattr(r, '__len__') else len(r), eng.last_timing(), flush=True)
rounds_single = eng.last_rounds()
me = DistRank(None, 1, 0, 0, st.cuda_stream, rmat=rm)
print("single relabeled", eng.relabeled(), eng.layout(), "dist relabeled", me.eng.relabeled(), me.eng.layout(), flush=True)
comm = TorchComm(); comm.bind_device(torch.device("cuda", 0))
for _ in range(3): stats, rec = run_rounds([me], comm, 1, True)
torch.cuda.synchronize(); e0.record(st)
for _ in range(5): stats, rec = run_rounds([me], comm, 1, True)
e1.record(st); torch.cuda.synchronize()
print("dist ms", e0.elapsed_time(e1) / 5, flush=True)
print("rounds single", len(rounds_single), "dist", len(stats))
for a, b in zip(rounds_single, stats):
    print(" ", (a.edges_before, a.edges_matched, a.edges_removed), (b.edges_before, b.edges_matched, b.edges_removed))
ms = mate.cpu().numpy(); md = me.mate.cpu().numpy()
print("mate equal", np.array_equal(ms, md), "matched single", int((ms >= 0).sum()), "dist", int((md >= 0).sum()))
dist.destroy_process_group()
