"""Where a one-rank run of the stepped multi-GPU protocol spends its time:
torch.profiler (CUPTI) over one matching; prints the kernel/collective table
and the host-side time of each protocol call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29541")
os.environ.setdefault("RANK", "0")
os.environ.setdefault("WORLD_SIZE", "1")
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1302_4587_b200 import dist as D  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
comm = D.TorchComm()
comm.bind_device(dev)
stream = torch.cuda.current_stream()
me = D.DistRank(None, 1, 0, 0, stream.cuda_stream,
                rmat=dict(scale=scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1, permute=True))
for _ in range(3):
    D.run_rounds([me], comm, 1, True)
torch.cuda.synchronize()

# host time per protocol call
calls = {}


def wrap(obj, name):
    f = getattr(obj, name)

    def g(*a, **k):
        t = time.perf_counter()
        r = f(*a, **k)
        calls.setdefault(name, [0.0, 0])
        calls[name][0] += time.perf_counter() - t
        calls[name][1] += 1
        return r
    setattr(obj, name, g)


for nm in ("round", "propose", "accept", "match", "hist", "begin"):
    wrap(me, nm)
for nm in ("alltoallv_stats", "allgather_bitmap", "allgather_mround", "allreduce_sum"):
    wrap(comm, nm)
t0 = time.perf_counter()
D.run_rounds([me], comm, 1, True)
torch.cuda.synchronize()
print(f"one matching wall {1e3 * (time.perf_counter() - t0):.2f} ms")
for k, (s, c) in sorted(calls.items(), key=lambda kv: -kv[1][0]):
    print(f"  host {k:18s} x{c:3d} {1e3 * s:8.2f} ms")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    D.run_rounds([me], comm, 1, True)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
dist.destroy_process_group()
