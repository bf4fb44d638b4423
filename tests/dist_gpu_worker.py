"""torchrun worker for tests/test_dist.py::test_two_processes_real_partitions.

TEST INFRASTRUCTURE.  Two processes, one liblmx partition each (the real
kernels: DistRank), talking through TorchComm over gloo -- the transport
code path of the NCCL runs, with the collectives staged through the host by
gloo.  Both processes share the one GPU of the test box: no kernel waits on
another rank (every exchange is a host-side gloo collective between two
complete launches), so the processes only time-slice the GPU.

Rank 0 checks every result against the pinned C oracle (matchers.py:61-122,
bsp.py:148-199 accounting) and the distributed RMAT build against the
single-GPU engine on lmx_gen_rmat's graph.
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1302_4587_b200 import Engine  # noqa: E402
from paper_1302_4587_b200.dist import (DistRank, TorchComm, _unpack_ids, build_rmat_distributed,  # noqa: E402
                                       round_messages, run_rounds)
from paper_1302_4587_b200.graph import Graph  # noqa: E402


def main():
    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    comm = TorchComm()
    comm.bind_device(dev)
    failures = 0
    cases = [(1, 300, 1200, "random"), (2, 257, 900, "ties"), (3, 64, 2000, "unit"), (4, 5000, 40000, "random")]
    for seed, n, m, kind in cases:
        rng = np.random.default_rng(seed)
        u = rng.integers(0, n, m)
        v = rng.integers(0, n, m)
        w = rng.random(m) if kind == "random" else (rng.integers(0, 3, m).astype(float) if kind == "ties"
                                                    else np.ones(m))
        gn, eu, ev, ew = O.build_graph_vec(u, v, w, n)
        g = Graph(gn, eu, ev, ew)
        for algo in ("compact", "auto"):
            me = DistRank(g, comm.p, comm.rank, 0, algo=algo)
            try:
                for rr in (True, False):
                    stats, records = run_rounds([me], comm, seed, rr)
                    msgs = round_messages([me], comm, len(stats))
                    mate, ebits = comm.gather_outputs([me])
                    if comm.rank == 0:
                        ids = _unpack_ids(ebits, me.m)
                        ref = O.c_local_max(gn, eu, ev, ew, seed, rr)
                        ok = (np.array_equal(mate.cpu().numpy()[:gn], ref.mate)
                              and np.array_equal(ids, ref.matched_ids)
                              and [(s.edges_before, s.edges_matched, s.edges_removed) for s in stats] == ref.rounds
                              and [tuple(vars(x).values()) if not isinstance(x, tuple) else x for x in msgs]
                              == O.bsp_messages(gn, eu, ev, ew, comm.p, seed, rr))
                        print(f"case seed={seed} n={n} kind={kind} algo={me.algo} rr={rr} rounds={len(stats)} "
                              f"cut-records={sum(records)} ok={ok}", flush=True)
                        failures += 0 if ok else 1
            finally:
                me.close()
    # the distributed RMAT builder (no rank holds the whole graph) over the
    # real transport, against the single-GPU engine on the same recipe
    for scale, permute in ((12, True), (14, False)):
        me = DistRank(None, comm.p, comm.rank, 0, defer=True)
        try:
            build_rmat_distributed([me], comm, scale, 16, 0.57, 0.19, 0.19, 3, permute, keep_records=True)
            stats, records = run_rounds([me], comm, 5, True)
            mate, ebits = comm.gather_outputs([me])
            # the multi-GPU e2e leg: the partition loads itself again from its
            # page-locked local edges and must give the same matching
            recs, k_local = me.host_records
            me.load_local_edges(recs, k_local, me.host_degrees, me.m)
            stats2, _ = run_rounds([me], comm, 5, True)
            mate2, ebits2 = comm.gather_outputs([me])
            same_again = stats2 == stats and torch.equal(mate2, mate) and torch.equal(ebits2, ebits)
            if comm.rank == 0:
                ids = _unpack_ids(ebits, me.m)
                with Engine(0) as eng:
                    eng.gen_rmat(scale, 16, 0.57, 0.19, 0.19, seed=3, permute=permute)
                    n1, m1 = eng.graph_size()
                    mate1, ids1, rounds1 = eng.match_raw(5, True)
                ok = (same_again and me.m == m1 and np.array_equal(mate.cpu().numpy()[:n1], mate1)
                      and np.array_equal(ids, ids1)
                      and [(s.edges_before, s.edges_matched, s.edges_removed) for s in stats]
                      == [(r.edges_before, r.edges_matched, r.edges_removed) for r in rounds1])
                print(f"rmat scale={scale} permute={permute} m={me.m} rounds={len(stats)} "
                      f"cut-records={sum(records)} ok={ok}", flush=True)
                failures += 0 if ok else 1
        finally:
            me.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(1 if failures else 0)


if __name__ == "__main__":
    main()
