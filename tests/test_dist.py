"""Multi-GPU (1D partition) path.

* CPU: world_size-2 torch.distributed (gloo) run of the real transport
  (``TorchComm``) and round protocol (``run_rounds``) over emulated partitions
  (tests/dist_emulator.py), checked against the oracle.
* GPU: ``local_max_dist`` (p liblmx partitions on one B200, the reference's
  logical-worker mode, bsp.py:13-16) must equal the single-GPU engine and the
  reference for every p (bsp.py:113-115; test_bsp.py:68-87).
"""

from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, instance_graph, mate_digest, small_cases, small_runs
from oracle import oracle as O


def _partition_cases():
    z = np.load(os.path.join(ROOT, "tests", "golden", "partition.npz"))
    for k in range(z["p"].size):
        kind, size, alpha, seed, p = (int(z[x][k]) for x in ("kind", "size", "alpha", "seed", "p"))
        n, eu, ev, w = O.gen_random(size, alpha, seed) if kind == 0 else O.gen_rgg(size, seed)
        b0 = int(z["boff"][k])
        yield n, eu, ev, w, p, z["bounds"][b0:b0 + p + 1], int(z["cut"][k]), float(z["imbalance"][k]), \
            float(z["cut_fraction"][k])


def test_partition_bounds_match_reference():
    """oracle.partition_bounds and the package's partition_graph (bsp.py:60-98
    mirror) vs the unmodified reference (tests/golden/partition.npz)."""
    from paper_1302_4587_b200 import Graph
    from paper_1302_4587_b200.dist import partition_graph
    for n, eu, ev, w, p, want, cut, imb, cf in _partition_cases():
        deg = np.bincount(np.concatenate([eu, ev]), minlength=n)
        offsets = np.concatenate([[0], np.cumsum(deg)])
        assert np.array_equal(O.partition_bounds(offsets, n, p), want)
        part = partition_graph(Graph(n, eu, ev, w), p)
        assert np.array_equal(part.bounds, want) and part.cut_edges.size == cut
        assert part.degree_imbalance == imb and part.cut_fraction == cf


def test_gloo_world_size_2_matches_oracle():
    env = dict(os.environ, OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517",
           os.path.join(ROOT, "tests", "dist_gloo_worker.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-4000:]
    assert out.count("ok=True") == 18 and "algo=scan" in out, out[-4000:]


@pytest.mark.gpu
def test_two_processes_real_partitions():
    """Two processes, each one liblmx partition (the real kernels), through
    TorchComm over gloo (tests/dist_gpu_worker.py): the multi-process path of
    the NCCL runs on the one GPU of the test box.  Matchings, RoundStats and
    RoundMessages against the C oracle; the distributed RMAT build against
    the single-GPU engine."""
    env = dict(os.environ, OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29519",
           os.path.join(ROOT, "tests", "dist_gpu_worker.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-4000:]
    assert out.count("ok=True") == 18 and "ok=False" not in out and "algo=scan" in out, out[-4000:]


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["auto", "compact"])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
def test_dist_equals_single_gpu_small(golden_small, p, algo):
    from paper_1302_4587_b200 import Graph
    from paper_1302_4587_b200.dist import local_max_dist
    graphs = {gi: (n, built) for gi, n, _, built, _ in small_cases(golden_small)}
    done = 0
    for gi, seed, rr, mate, ids, rounds in small_runs(golden_small):
        n, (eu, ev, w) = graphs[gi]
        if n < p or gi % 7:   # a spread of cases; each run sets up p contexts
            continue
        matching, trace = local_max_dist(Graph(n, eu, ev, w), p, seed, rr, algo=algo)
        assert np.array_equal(matching.mate, mate), (gi, seed, rr, p)
        assert np.array_equal(matching.sorted_edge_ids(), ids), (gi, seed, rr, p)
        assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in trace.rounds] == rounds
        done += 1
    assert done > 20


@pytest.mark.gpu
@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("name", ["random-x16-a4-wunit-s0", "rgg-x16-euclidean-s0", "random-x12-a16-s5",
                                  "delaunay_x10"])
def test_dist_reference_instances(golden_instances, name, p):
    from paper_1302_4587_b200 import Graph
    from paper_1302_4587_b200.dist import local_max_dist
    z = golden_instances
    n, eu, ev, w = instance_graph(z, name)
    matching, trace = local_max_dist(Graph(n, eu, ev, w), p, int(z[f"{name}/seed"]), bool(z[f"{name}/rerandomize"]))
    assert mate_digest(matching.mate) == str(z[f"{name}/mate_digest"])
    assert [[r.edges_before, r.edges_matched, r.edges_removed] for r in trace.rounds] == \
        z[f"{name}/rounds"].tolist()
    assert sum(m.candidate_records for m in trace.messages) > 0 and sum(trace.exchange_a_records) > 0


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["auto", "compact"])
def test_dist_rmat_skewed_equals_single(engine, algo):
    """RMAT (relabelled, hubs) split over 4 partitions equals the single-GPU run."""
    from paper_1302_4587_b200.dist import local_max_dist
    engine.gen_rmat(14, 16, seed=5)
    g = engine.export_graph()
    mate, ids, rounds = engine.match_raw(5, True)
    matching, trace = local_max_dist(g, 4, 5, True, algo=algo)
    assert np.array_equal(matching.mate, mate)
    assert np.array_equal(matching.sorted_edge_ids(), ids)
    assert trace.rounds == rounds


@pytest.mark.gpu
def test_run_matcher_dist_engine():
    from paper_1302_4587_b200 import Graph, run_matcher
    n, eu, ev, w = O.gen_random(1 << 10, 4, 2)
    g = Graph(n, eu, ev, w)
    a, _ = run_matcher(g, "localmax", 2, engine="b200")
    b, _ = run_matcher(g, "localmax", 2, engine="b200-dist", p=3)
    assert a == b


@pytest.mark.gpu
def test_dist_round_loop_choice():
    """Distinct weights put the partitions on the scan loop; ties on the compacting loop."""
    from paper_1302_4587_b200 import Graph
    from paper_1302_4587_b200.dist import DistRank
    n, eu, ev, w = O.gen_random(1 << 9, 4, 3)
    for weights, want in ((w, "scan"), (np.ones_like(w), "compact")):
        r = DistRank(Graph(n, eu, ev, weights), 2, 1)
        try:
            assert r.algo == want
        finally:
            r.close()


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["auto", "compact"])
def test_dist_round_messages_equal_reference(algo):
    """trace.messages of local_max_dist == the unmodified reference's
    bsp_local_max RoundMessages (tests/golden/bsp.npz), field by field, and
    the partitions own exactly partition_graph's ranges."""
    from paper_1302_4587_b200 import Graph
    from paper_1302_4587_b200.dist import DistRank, local_max_dist
    z = np.load(os.path.join(ROOT, "tests", "golden", "bsp.npz"))
    for k, (kind, size, alpha, seed, p, rr) in enumerate(z["cases"]):
        n, eu, ev, w = O.gen_random(int(size), int(alpha), int(seed)) if kind == 0 else O.gen_rgg(int(size), int(seed))
        g = Graph(n, eu, ev, w)
        _, trace = local_max_dist(g, int(p), int(seed), bool(rr), algo=algo)
        want = [tuple(int(x) for x in row) for row in z["rows"][z["off"][k]:z["off"][k + 1]]]
        got = [(m.round_index, m.candidate_records, m.bytes_estimate, m.cut_edges_surviving, m.status_records)
               for m in trace.messages]
        assert got == want, (k, got[:3], want[:3])
        if p > 1 and k % 5 == 0:
            deg = np.bincount(np.concatenate([eu, ev]), minlength=n)
            r = DistRank(g, int(p), 0, algo=algo)
            try:
                assert np.array_equal(r.bounds, O.partition_bounds(np.concatenate([[0], np.cumsum(deg)]), n, int(p)))
            finally:
                r.close()


@pytest.mark.gpu
def test_partition_memory_shrinks_with_p():
    """A partition keeps its local edges and owned slots only: device bytes per
    rank fall roughly as 1/p (global bitmaps and per-vertex arrays aside)."""
    from paper_1302_4587_b200 import Engine
    from paper_1302_4587_b200.dist import DistRank
    eng = Engine(0)
    eng.gen_rmat(20, 16, seed=3)
    g = eng.export_graph()
    eng.close()
    per = {}
    for p in (1, 2, 4):
        r = DistRank(g, p, p - 1)
        try:
            per[p] = r.eng.device_bytes()
        finally:
            r.close()
    assert per[2] < 0.8 * per[1] and per[4] < 0.65 * per[1], per


@pytest.mark.gpu
def test_reference_bsp_assertions_with_b200_engine():
    """test_bsp.py:59-98 with bsp_local_max replaced by local_max_dist."""
    from paper_1302_4587_b200 import Graph, local_max_b200, validate_matching
    from paper_1302_4587_b200.dist import local_max_dist, partition_graph
    n, eu, ev, w = O.gen_random(256, 4, 2)
    g = Graph(n, eu, ev, w)
    base, _ = local_max_b200(g, 9)
    matching, trace = local_max_dist(g, 1, 9)
    assert matching == base
    assert all(rm.candidate_records == 0 for rm in trace.messages)
    assert all(rm.bytes_estimate == 0 for rm in trace.messages)
    n, eu, ev, w = O.gen_rgg(12, 4)
    g = Graph(n, eu, ev, w)
    base, _ = local_max_b200(g, 7)
    for p in (2, 4, 8):
        matching, trace = local_max_dist(g, p, 7)
        assert matching == base
        check = validate_matching(g, matching)
        assert check.valid and check.maximal
    n, eu, ev, w = O.gen_random(256, 4, 6)
    unit = Graph(n, eu, ev, np.ones_like(w))
    base, _ = local_max_b200(unit, 3)
    for p in (1, 2, 4, 8):
        matching, _ = local_max_dist(unit, p, 3)
        assert matching == base
    n, eu, ev, w = O.gen_random(512, 4, 8)
    _, trace = local_max_dist(Graph(n, eu, ev, w), 8, 1)
    for rm in trace.messages:
        assert rm.candidate_records <= 2 * rm.cut_edges_surviving
        assert rm.bytes_estimate == rm.candidate_records * 32
    cuts = [rm.cut_edges_surviving for rm in trace.messages]
    assert cuts == sorted(cuts, reverse=True)
    n1, eu1, ev1, w1 = O.gen_rgg(12, 5)
    alpha = max(1, round(len(eu1) / 4096))
    n2, eu2, ev2, w2 = O.gen_random(4096, alpha, 5)
    assert partition_graph(Graph(n1, eu1, ev1, w1), 8).cut_fraction < \
        partition_graph(Graph(n2, eu2, ev2, w2), 8).cut_fraction


@pytest.mark.gpu
@pytest.mark.parametrize("p", [2, 3, 4])
@pytest.mark.parametrize("scale,permute", [(12, True), (15, True), (14, False)])
def test_distributed_rmat_build_equals_single_gpu(engine, p, scale, permute):
    """The distributed builder (every rank keeps the pairs of its build range,
    bitmaps + degrees summed, records routed to the owners) gives the same
    graph: the matching, RoundStats and edge count equal the single-GPU run on
    lmx_gen_rmat's graph."""
    from paper_1302_4587_b200.dist import local_max_dist_rmat
    engine.gen_rmat(scale, 16, 0.57, 0.19, 0.19, seed=3, permute=permute)
    n, m = engine.graph_size()
    mate, ids, rounds = engine.match_raw(5, True)
    matching, trace, dev_bytes = local_max_dist_rmat(p, scale, 5, True, graph_seed=3, permute=permute)
    assert np.array_equal(np.asarray(matching.mate), mate)
    assert np.array_equal(matching.sorted_edge_ids(), ids)
    assert trace.rounds == rounds and rounds[0].edges_before == m
    assert len(dev_bytes) == p


@pytest.mark.gpu
@pytest.mark.parametrize("p", [2, 3])
def test_partition_reload_from_host_records(p):
    """The multi-GPU end-to-end leg (bench.py --gpus N): every partition kept
    its local edges (with global ids) in page-locked host memory at build
    time and loads itself again from them (DistRank.load_local_edges); the
    matching, RoundStats and gathered mate equal the first load's."""
    import torch
    from paper_1302_4587_b200.dist import DistRank, LocalComm, _unpack_ids, build_rmat_distributed, run_rounds
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream(0).cuda_stream
    ranks = [DistRank(None, p, k, 0, stream, defer=True) for k in range(p)]
    try:
        comm = LocalComm(p)
        build_rmat_distributed(ranks, comm, 13, 16, 0.57, 0.19, 0.19, 7, True, keep_records=True)
        stats0, _ = run_rounds(ranks, comm, 5, True)
        mate0, eb0 = comm.gather_outputs(ranks)
        mate0, ids0 = mate0.cpu().numpy().copy(), _unpack_ids(eb0, ranks[0].m)
        for _ in range(2):
            for r in ranks:
                recs, k = r.host_records
                r.load_local_edges(recs, k, r.host_degrees, r.m)
            stats1, _ = run_rounds(ranks, comm, 5, True)
            mate1, eb1 = comm.gather_outputs(ranks)
            assert stats1 == stats0
            assert np.array_equal(mate1.cpu().numpy(), mate0)
            assert np.array_equal(_unpack_ids(eb1, ranks[0].m), ids0)
    finally:
        for r in ranks:
            r.close()
