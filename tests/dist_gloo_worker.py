"""torchrun worker for tests/test_dist.py: TorchComm over gloo, world_size 2,
with the CPU partition emulator; rank 0 checks the result against the oracle."""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from dist_emulator import EmulatedRank  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1302_4587_b200.dist import TorchComm, _unpack_ids, round_messages, run_rounds  # noqa: E402
from paper_1302_4587_b200.graph import Graph  # noqa: E402


def main():
    dist.init_process_group("gloo")
    comm = TorchComm()
    comm.bind_device(torch.device("cpu"))
    failures = 0
    cases = [(1, 300, 1200, "random"), (2, 257, 900, "ties"), (3, 64, 2000, "unit"), (4, 500, 400, "random")]
    for seed, n, m, kind in cases:
        rng = np.random.default_rng(seed)
        u = rng.integers(0, n, m)
        v = rng.integers(0, n, m)
        w = rng.random(m) if kind == "random" else (rng.integers(0, 3, m).astype(float) if kind == "ties"
                                                    else np.ones(m))
        gn, eu, ev, ew = O.build_graph_vec(u, v, w, n)
        g = Graph(gn, eu, ev, ew)
        for algo, rr in (("compact", True), ("compact", False), ("scan", True), ("scan", False)):
            me = EmulatedRank(g, comm.p, comm.rank, algo)
            stats, records = run_rounds([me], comm, seed, rr)
            msgs = round_messages([me], comm, len(stats))
            mate, ebits = comm.gather_outputs([me])
            if comm.rank == 0:
                ids = _unpack_ids(ebits, me.m)
                ref = O.c_local_max(gn, eu, ev, ew, seed, rr)
                ok = (np.array_equal(mate.numpy()[:gn], ref.mate) and np.array_equal(ids, ref.matched_ids)
                      and [(s.edges_before, s.edges_matched, s.edges_removed) for s in stats] == ref.rounds
                      and [tuple(vars(x).values()) if not isinstance(x, tuple) else x for x in msgs]
                      == O.bsp_messages(gn, eu, ev, ew, comm.p, seed, rr))
                print(f"case seed={seed} n={n} kind={kind} algo={algo} rr={rr} rounds={len(stats)} "
                      f"cut-records={sum(records)} ok={ok}", flush=True)
                failures += 0 if ok else 1
    # the distributed builder's collectives (TorchComm side) on CPU tensors
    class _R:
        device = torch.device("cpu")
    me = _R()
    t = torch.tensor([1 << (3 * comm.rank), 7 + comm.rank], dtype=torch.int32)
    comm.allreduce_sum_([me], [t])
    lo = comm.allreduce_min_u64([me], [torch.tensor([100 + comm.rank], dtype=torch.int64)])
    hi = comm.allreduce_max_u64([me], [torch.tensor([100 + comm.rank], dtype=torch.int64)])
    # rank k sends k + 1 records of width 6 to every rank
    counts = np.array([comm.rank + 1] * comm.p, dtype=np.int64)
    send = torch.arange(int(counts.sum()) * 6, dtype=torch.int32).reshape(-1, 6) + 1000 * comm.rank
    box = {}

    def recv_buffer(r, cnt):
        box["buf"] = torch.zeros((max(cnt, 1), 6), dtype=torch.int32)
        return box["buf"]
    (got,) = comm.alltoallv_records([me], [(send, counts)], 6, recv_buffer)
    want_total = sum(k + 1 for k in range(comm.p))
    ok = (t.tolist() == [1 + 8, 7 + 8] and lo == 100 and hi == 100 + comm.p - 1 and got == want_total
          and int(box["buf"][0, 0]) == 6 * (comm.rank * 1))
    print(f"collectives rank={comm.rank} ok={ok}", flush=True)
    failures += 0 if ok else 1
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(1 if failures else 0)


if __name__ == "__main__":
    main()
