"""Parity of the sm_100a engine with the reference (golden fixtures) and the
pinned CPU oracle.  Bar: bit-exact mate arrays, matched id sets and RoundStats
traces (integer work), as the reference's own engine-equivalence tests demand
(test_pram.py:164-176, 219-236; test_bsp.py:68-87)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import edges_digest, instance_graph, mate_digest, small_cases, small_runs
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _graph(n, eu, ev, w):
    from paper_1302_4587_b200 import Graph
    return Graph(n, eu, ev, w)


# (weight-key layout, relabelling, round loop): the scan loop serves the
# distinct layout by default; the compacting loop is forced on it as well.
VARIANTS = [("auto", "auto", "auto"), ("distinct", "on", "scan"), ("distinct", "off", "compact"),
            ("distinct", "off", "scan"), ("general", "off", "auto"), ("general", "on", "auto")]


@pytest.fixture(params=VARIANTS, ids=lambda p: f"{p[0]}-relabel_{p[1]}-{p[2]}")
def layout_engine(engine, request):
    """The engine with a forced weight-key layout, relabelling mode and round loop."""
    engine.set_layout(request.param[0])
    engine.set_relabel(request.param[1])
    engine.set_algo(request.param[2])
    yield engine
    engine.set_layout("auto")
    engine.set_relabel("auto")
    engine.set_algo("auto")


def test_small_golden_runs_bit_exact(layout_engine, golden_small):
    """~1600 reference runs on 409 small graphs: ties, -0.0, zero weights,
    edgeless graphs, both rerandomize settings -- under every weight layout."""
    engine = layout_engine
    graphs = {gi: (n, built) for gi, n, _, built, _ in small_cases(golden_small)}
    loaded = None
    count = 0
    for gi, seed, rr, mate, ids, rounds in small_runs(golden_small):
        n, (eu, ev, w) = graphs[gi]
        g = _graph(n, eu, ev, w)
        if loaded != gi:
            engine.load_graph(g)
            loaded = gi
        matching, trace = engine.match(g, seed, rr)
        assert np.array_equal(matching.mate, mate), (gi, seed, rr)
        assert np.array_equal(matching.sorted_edge_ids(), ids), (gi, seed, rr)
        assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in trace.rounds] == rounds, \
            (gi, seed, rr)
        count += 1
    assert count > 1000


@pytest.mark.parametrize("name", [
    "random-x16-a4-wunit-s0", "random-x16-a4-wunit-s0-norr", "random-x16-a4-s0",
    "rgg-x16-euclidean-s0", "rgg-x12-random-s3", "random-x12-a16-s5",
    "random-x10-a200-dense-s1", "delaunay_x10", "delaunay_x10-unit",
    "random-x20-a4-s1", "random-x20-a4-wunit-s2"])
def test_reference_instances_bit_exact(engine, golden_instances, name):
    z = golden_instances
    n, eu, ev, w = instance_graph(z, name)
    assert edges_digest(eu, ev, w) == str(z[f"{name}/edges_sha"])
    g = _graph(n, eu, ev, w)
    engine.load_graph(g)
    matching, trace = engine.match(g, int(z[f"{name}/seed"]), bool(z[f"{name}/rerandomize"]))
    assert mate_digest(matching.mate) == str(z[f"{name}/mate_digest"])
    if f"{name}/mate" in z:
        assert np.array_equal(matching.mate, z[f"{name}/mate"].astype(np.int64))
    assert [[r.edges_before, r.edges_matched, r.edges_removed] for r in trace.rounds] == \
        z[f"{name}/rounds"].tolist()
    assert matching.size == int(z[f"{name}/size"])
    assert matching.weight(g) == float(z[f"{name}/weight"])


def test_drop_in_entry_point_c1():
    """local_max_b200 with the local_max_seq contract on config C1."""
    from paper_1302_4587_b200 import local_max_b200, validate_matching
    n, eu, ev, w = O.gen_random(1 << 16, 4, 0, unit=True)
    g = _graph(n, eu, ev, w)
    matching, trace = local_max_b200(g, 0)
    assert matching.size == 29214
    assert trace.total_rounds == 5
    assert mate_digest(matching.mate) == "34039b07576f826f"
    chk = validate_matching(g, matching)
    assert chk.valid and chk.maximal


def test_random_graphs_vs_oracle(layout_engine):
    engine = layout_engine
    rng = np.random.default_rng(7)
    for trial in range(60):
        n = int(rng.integers(2, 3000))
        m = int(rng.integers(0, 8 * n))
        u = rng.integers(0, n, m)
        v = rng.integers(0, n, m)
        mode = trial % 3
        w = rng.random(m) if mode == 0 else (rng.integers(0, 3, m).astype(float) if mode == 1 else np.ones(m))
        gn, eu, ev, ew = O.build_graph_vec(u, v, w, n)
        g = _graph(gn, eu, ev, ew)
        engine.load_graph(g)
        for seed, rr in ((trial, True), (trial + 1, False)):
            res = O.c_local_max(gn, eu, ev, ew, seed, rr)
            matching, trace = engine.match(g, seed, rr)
            assert np.array_equal(matching.mate, res.mate), (trial, seed)
            assert np.array_equal(matching.sorted_edge_ids(), res.matched_ids)
            assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in trace.rounds] == res.rounds


def test_hubs_and_skew_vs_oracle(layout_engine):
    """Stars and skewed degrees exercise every bucket mapping (thread, 8-lane
    group, warp, block; degrees around each threshold) including multi-pass
    in-place hub compaction."""
    engine = layout_engine
    rng = np.random.default_rng(11)
    parts_u, parts_v = [], []
    n = 60000
    for hub, deg in ((0, 50000), (1, 32768), (2, 32767), (3, 1025), (4, 1024), (5, 300), (6, 33)):
        nb = rng.choice(np.arange(7, n), size=deg, replace=False)
        parts_u.append(np.full(deg, hub))
        parts_v.append(nb)
    parts_u.append(rng.integers(7, n, 200000))
    parts_v.append(rng.integers(7, n, 200000))
    u = np.concatenate(parts_u)
    v = np.concatenate(parts_v)
    for mode in range(3):
        w = rng.random(u.size) if mode == 0 else (np.ones(u.size) if mode == 1 else rng.integers(0, 4, u.size) * 0.5)
        gn, eu, ev, ew = O.build_graph_vec(u, v, w, n)
        g = _graph(gn, eu, ev, ew)
        engine.load_graph(g)
        for seed in (0, 5):
            res = O.c_local_max(gn, eu, ev, ew, seed, True)
            matching, trace = engine.match(g, seed, True)
            assert np.array_equal(matching.mate, res.mate), (mode, seed)
            assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in trace.rounds] == res.rounds


def test_rerun_on_same_graph_is_identical(engine):
    n, eu, ev, w = O.gen_random(1 << 14, 8, 3)
    g = _graph(n, eu, ev, w)
    engine.load_graph(g)
    a, ta = engine.match(g, 9)
    b, tb = engine.match(g, 9)
    c, _ = engine.match(g, 10)
    assert a == b and ta.rounds == tb.rounds
    res = O.c_local_max(n, eu, ev, w, 10)
    assert np.array_equal(c.mate, res.mate)


def test_long_chain_many_rounds(engine):
    """A path with increasing weights and rerandomize off needs ~m/2 rounds
    (local max matches one edge per round from the heavy end)."""
    m = 3000
    eu = np.arange(m, dtype=np.int64)
    ev = eu + 1
    w = np.arange(m, dtype=np.float64)
    g = _graph(m + 1, eu, ev, w)
    engine.load_graph(g)
    res = O.c_local_max(m + 1, eu, ev, w, 0, False)
    matching, trace = engine.match(g, 0, False)
    assert len(res.rounds) > 1000
    assert np.array_equal(matching.mate, res.mate)
    assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in trace.rounds] == res.rounds


@pytest.mark.parametrize("m", [6, 28, 40, 300, 520])
@pytest.mark.parametrize("algo", ["scan", "compact"])
def test_chains_across_round_count_regimes(engine, m, algo):
    """Paths with increasing weights: ~m/2 rounds, so the scan loop's death-round
    histogram runs with 4-bit (< 15 rounds), 8-bit (< 255) and 32-bit round
    codes; the compacting loop on the same graphs."""
    eu = np.arange(m, dtype=np.int64)
    ev = eu + 1
    w = np.arange(m, dtype=np.float64)
    g = _graph(m + 1, eu, ev, w)
    engine.set_algo(algo)
    try:
        engine.load_graph(g)
        assert engine.algo() == algo
        for rr in (False, True):
            res = O.c_local_max(m + 1, eu, ev, w, 3, rr)
            matching, trace = engine.match(g, 3, rr)
            assert np.array_equal(matching.mate, res.mate)
            assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in trace.rounds] == res.rounds
    finally:
        engine.set_algo("auto")


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_scan_loop_ties_and_rerandomize(engine, seed):
    """Distinct layout with tied weight groups (so tied runs inside the weight-
    ordered segments are resolved by the per-round salt), both rerandomize
    modes, scan loop against the oracle and against the compacting loop."""
    rng = np.random.default_rng(seed)
    n = 3000
    _, eu, ev, _ = O.gen_random(n, 8, seed)
    m = eu.size
    w = rng.random(m)
    tied = rng.random(m) < 0.05           # 5% of the edges share a few weights
    w[tied] = rng.choice([0.25, 0.5, 0.75], size=int(tied.sum()))
    g = _graph(n, eu, ev, w)
    outs = {}
    for algo in ("scan", "compact"):
        engine.set_algo(algo)
        engine.set_layout("distinct")
        try:
            engine.load_graph(g)
            assert engine.algo() == algo and engine.layout() == "distinct"
            for rr in (True, False):
                res = O.c_local_max(n, eu, ev, w, seed, rr)
                matching, trace = engine.match(g, seed, rr)
                assert np.array_equal(matching.mate, res.mate)
                assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in trace.rounds] == res.rounds
                outs[(algo, rr)] = matching.mate.copy()
        finally:
            engine.set_algo("auto")
            engine.set_layout("auto")
    assert np.array_equal(outs[("scan", True)], outs[("compact", True)])


def test_domain_errors_raise_value_error(engine):
    from paper_1302_4587_b200 import local_max_b200
    bad = [
        (3, [0, 1], [1, 2], [1.0, -1.0]),
        (3, [0, 1], [1, 2], [1.0, float("nan")]),
        (3, [0, 1], [1, 2], [float("inf"), 1.0]),
        (3, [0, 1], [1, 3], [1.0, 1.0]),
        (3, [0, -1], [1, 2], [1.0, 1.0]),
        (3, [0, 1], [1, 1], [1.0, 1.0]),
    ]
    for n, u, v, w in bad:
        g = _graph(n, np.array(u), np.array(v), np.array(w))
        with pytest.raises(ValueError):
            local_max_b200(g, 0)


def test_empty_and_edgeless(engine):
    for n in (0, 1, 5):
        g = _graph(n, np.empty(0, np.int64), np.empty(0, np.int64), np.empty(0))
        engine.load_graph(g)
        matching, trace = engine.match(g, 3)
        assert matching.size == 0 and trace.total_rounds == 0
        assert np.array_equal(matching.mate, np.full(n, -1))


def test_device_build_graph_matches_reference_numbering(golden_small):
    from paper_1302_4587_b200 import build_graph
    for gi, n, raw, built, nv in small_cases(golden_small):
        g = build_graph(tuple(raw), nv)
        assert g.num_vertices == n, gi
        assert np.array_equal(g.edge_u, built[0]) and np.array_equal(g.edge_v, built[1]), gi
        assert np.array_equal(g.edge_weight.view(np.uint64), built[2].view(np.uint64)), gi


def test_device_build_graph_errors():
    from paper_1302_4587_b200 import build_graph
    with pytest.raises(ValueError, match="edge 1"):
        build_graph([(0, 1, 1.0), (0, -2, 1.0)])
    with pytest.raises(ValueError, match="out of range"):
        build_graph([(0, 1, 1.0), (0, 5, 1.0)], num_vertices=3)
    with pytest.raises(ValueError, match="weight"):
        build_graph([(0, 1, float("nan"))])


def test_layout_selection(engine):
    n, eu, ev, w = O.gen_random(1 << 10, 4, 1)
    engine.load_graph(_graph(n, eu, ev, w))
    assert engine.layout() == "distinct"
    engine.load_graph(_graph(n, eu, ev, np.ones_like(w)))
    assert engine.layout() == "uniform"
    engine.load_graph(_graph(n, eu, ev, np.floor(w * 3)))
    assert engine.layout() == "general"
    assert not engine.relabeled()          # ER degrees are not skewed
    engine.gen_rmat(14, 16, seed=3)
    assert engine.relabeled()              # RMAT is


def test_rmat_generator_matches_oracle(engine):
    for scale, ef, seed, perm in ((10, 16, 1, True), (12, 8, 7, False), (14, 16, 2, True)):
        u, v, w = engine.gen_rmat_raw(scale, ef, seed=seed, permute=perm)
        ou, ov, ow = O.rmat_raw(scale, ef, seed=seed, permute=perm)
        assert np.array_equal(u, ou) and np.array_equal(v, ov)
        assert np.array_equal(w.view(np.uint64), ow.view(np.uint64))
        engine.gen_rmat(scale, ef, seed=seed, permute=perm)
        g = engine.export_graph()
        n, eu, ev, ew = O.build_graph_vec(ou, ov, ow, 1 << scale)
        assert g.num_vertices == n
        assert np.array_equal(g.edge_u, eu) and np.array_equal(g.edge_v, ev)
        assert np.array_equal(g.edge_weight, ew)
        res = O.c_local_max(n, eu, ev, ew, seed, True)
        mate, ids, rounds = engine.match_raw(seed, True)
        assert np.array_equal(mate, res.mate)
        assert np.array_equal(ids, res.matched_ids)
        assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in rounds] == res.rounds


@pytest.mark.slow
def test_rmat20_vs_oracle(engine):
    """RMAT scale 20 (≈16 M edges, hubs > 10^4): full parity with the C oracle."""
    engine.gen_rmat(20, 16, seed=1, permute=True)
    g = engine.export_graph()
    res = O.c_local_max(g.num_vertices, g.edge_u, g.edge_v, g.edge_weight, 1, True)
    mate, ids, rounds = engine.match_raw(1, True)
    assert np.array_equal(mate, res.mate)
    assert np.array_equal(ids, res.matched_ids)
    assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in rounds] == res.rounds


@pytest.mark.gpu
def test_scan_speculative_batch_across_round_counts(engine):
    """A repeated matching of one loaded graph enqueues its first batch from the
    previous round count (one synchronisation).  Tied pairs on a decreasing
    path make the round count depend on the seed (2 .. 8 rounds without
    rerandomize), so later seeds run past the speculated batch, and shorter
    ones end inside it; every result equals the oracle."""
    n = 30
    eu = np.arange(n - 1, dtype=np.int64)
    ev = eu + 1
    w = np.repeat(np.arange(40)[::-1].astype(np.float64) + 1.0, 2)[: n - 1]
    g = _graph(n, eu, ev, w)
    engine.set_algo("scan")
    engine.set_layout("distinct")
    try:
        engine.load_graph(g)
        assert engine.algo() == "scan"
        counts = []
        for seed in (14, 0, 1, 3, 15, 0, 14, 4):
            res = O.c_local_max(n, eu, ev, w, seed, False)
            matching, trace = engine.match(g, seed, False)
            assert np.array_equal(matching.mate, res.mate), seed
            assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in trace.rounds] == res.rounds
            counts.append(len(res.rounds))
        assert max(b - a for a, b in zip(counts, counts[1:])) >= 2
    finally:
        engine.set_algo("auto")
        engine.set_layout("auto")
