"""rerandomize=False on tied weights through the static (weight, salt) layout
(LMX_OPT_STATIC_ORDER): with rerandomize off every round's salts are round
0's (tiebreak.py:40-52), so the key order is fixed for the run and the
weight-ordered scan loop serves unit / tie-heavy weights.  Results must equal
the reference's local_max_seq(g, seed, rerandomize=False) bit for bit."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import instance_graph, mate_digest, small_cases, small_runs
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _graph(n, eu, ev, w):
    from paper_1302_4587_b200 import Graph
    return Graph(n, eu, ev, w)


def test_small_golden_runs_static(engine, golden_small):
    """every rerandomize=False reference run of the small goldens (ties, -0.0,
    zero weights, edgeless graphs), each graph laid out for its run's seed"""
    graphs = {gi: (n, built) for gi, n, _, built, _ in small_cases(golden_small)}
    count = static = 0
    for gi, seed, rr, mate, ids, rounds in small_runs(golden_small):
        if rr:
            continue
        n, (eu, ev, w) = graphs[gi]
        g = _graph(n, eu, ev, w)
        engine.set_static_order(seed)
        engine.load_graph(g)
        static += engine.static_order()
        matching, trace = engine.match(g, seed, False)
        assert np.array_equal(matching.mate, mate), (gi, seed)
        assert np.array_equal(matching.sorted_edge_ids(), ids), (gi, seed)
        assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in trace.rounds] == rounds, (gi, seed)
        count += 1
    engine.set_static_order(None)
    assert count > 300 and static > 100


@pytest.mark.parametrize("kind", ["unit", "three", "rgg"])
@pytest.mark.parametrize("seed", [0, 7, -1, (1 << 64) + 7])
def test_static_vs_oracle(engine, kind, seed):
    if kind == "rgg":
        n, eu, ev, w = O.gen_rgg(13, 2)
        w = np.round(w * 20) / 20                          # many ties
    else:
        n, eu, ev, w = O.gen_random(30_000, 8, 11, unit=(kind == "unit"))
        if kind == "three":
            w = np.floor(w * 3)                            # three distinct values
    ref = O.c_local_max(n, eu, ev, w, seed, False)
    engine.set_static_order(seed)
    engine.load_graph(_graph(n, eu, ev, w))
    engine.set_static_order(None)
    assert engine.static_order() and engine.algo() == "scan"
    mate, ids, rounds = engine.match_raw(seed, False)
    assert np.array_equal(mate, ref.mate) and np.array_equal(ids, ref.matched_ids)
    assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in rounds] == ref.rounds
    again = engine.match_raw(seed, False)                  # repeatable on the same layout
    assert np.array_equal(again[0], mate)
    # the layout serves exactly that seed, without rerandomisation
    with pytest.raises(RuntimeError, match="static|fixed salt order"):
        engine.match_raw(seed + 1, False)
    with pytest.raises(RuntimeError, match="static|fixed salt order"):
        engine.match_raw(seed, True)


def test_distinct_weights_ignore_static(engine):
    n, eu, ev, w = O.gen_random(20_000, 6, 4)
    engine.set_static_order(3)
    engine.load_graph(_graph(n, eu, ev, w))
    engine.set_static_order(None)
    assert not engine.static_order()                       # no ties: the ordinary layout serves any seed
    for seed, rr in ((3, False), (9, True)):
        ref = O.c_local_max(n, eu, ev, w, seed, rr)
        mate, ids, _ = engine.match_raw(seed, rr)
        assert np.array_equal(mate, ref.mate) and np.array_equal(ids, ref.matched_ids)


def test_drop_in_uses_static_layout(golden_instances):
    """local_max_b200(g, seed, rerandomize=False) on unit weights takes the
    static layout; the reference instance's digest is unchanged"""
    from paper_1302_4587_b200 import local_max_b200
    from paper_1302_4587_b200.engine import default_engine
    z = golden_instances
    name = "random-x16-a4-wunit-s0-norr"
    n, eu, ev, w = instance_graph(z, name)
    assert not bool(z[f"{name}/rerandomize"])
    g = _graph(n, eu, ev, w)
    matching, trace = local_max_b200(g, int(z[f"{name}/seed"]), False)
    assert default_engine().static_order()
    assert mate_digest(matching.mate) == str(z[f"{name}/mate_digest"])
    assert [[r.edges_before, r.edges_matched, r.edges_removed] for r in trace.rounds] == \
        z[f"{name}/rounds"].tolist()
    matching2, _ = local_max_b200(g, 5, True)              # the next call reloads without it
    assert not default_engine().static_order()
    ref = O.c_local_max(n, eu, ev, w, 5, True)
    assert np.array_equal(matching2.mate, ref.mate)


def test_one_shot_entry_static(golden_instances):
    """lmx_local_max (the INTEGRATION.md entry) with rerandomize=0 on unit weights"""
    import ctypes

    from paper_1302_4587_b200 import load_library
    lib = load_library()
    z = golden_instances
    name = "random-x16-a4-wunit-s0-norr"
    n, eu, ev, w = instance_graph(z, name)
    seed = int(z[f"{name}/seed"])
    m = len(eu)
    mate = np.empty(n, dtype=np.int64)
    ids = np.empty(n // 2 + 1, dtype=np.int64)
    nm = ctypes.c_int64()
    nr = ctypes.c_int()
    rounds = np.empty(4096 * 3, dtype=np.int64)
    err = ctypes.create_string_buffer(512)
    eu = np.ascontiguousarray(eu, dtype=np.int64)
    ev = np.ascontiguousarray(ev, dtype=np.int64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    rc = lib.lmx_local_max(0, n, m, eu.ctypes.data, ev.ctypes.data, w.ctypes.data,
                           ctypes.c_uint64(seed & ((1 << 64) - 1)), 0, mate.ctypes.data, ids.ctypes.data,
                           ctypes.byref(nm), rounds.ctypes.data, 4096, ctypes.byref(nr), err, 512)
    assert rc == 0, err.value
    assert mate_digest(mate) == str(z[f"{name}/mate_digest"])
    assert rounds[:3 * nr.value].reshape(-1, 3).tolist() == z[f"{name}/rounds"].tolist()
