"""Property-based parity: random small graphs -- few distinct weights (ties),
zero and -0.0 weights, hubs, isolated vertices, both rerandomize settings,
seeds across the u64 range -- through every engine path (auto, forced
compacting loop, forced scan loop, static order, host and device loads)
against the pinned C oracle of matchers.py:61-122."""

from __future__ import annotations

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@st.composite
def graphs(draw):
    n = draw(st.integers(2, 300))
    k = draw(st.integers(0, 3 * n))
    rng = np.random.default_rng(draw(st.integers(0, 2**32 - 1)))
    hub = draw(st.booleans())
    u = rng.integers(0, n, size=k)
    v = rng.integers(0, n, size=k)
    if hub and k:
        u[: k // 2] = 0                                      # a hub at vertex 0
    palette = draw(st.sampled_from(["distinct", "few", "unit", "zeros"]))
    if palette == "distinct":
        w = rng.random(k)
    elif palette == "few":
        w = rng.integers(0, 4, size=k).astype(np.float64) / 2.0
    elif palette == "unit":
        w = np.ones(k)
    else:
        w = np.where(rng.random(k) < 0.5, 0.0, -0.0) + (rng.random(k) < 0.2)
    n2, eu, ev, ew = O.build_graph_vec(u, v, w, n)
    seed = draw(st.one_of(st.integers(0, 2**64 - 1), st.integers(-2**63, -1)))
    rr = draw(st.booleans())
    return n2, eu, ev, ew, seed, rr


def _graph(n, eu, ev, w):
    from paper_1302_4587_b200 import Graph
    return Graph(n, eu, ev, w)


@settings(max_examples=400, deadline=None, suppress_health_check=list(HealthCheck))
@given(graphs(), st.sampled_from(["auto", "compact", "scan", "static", "device"]))
def test_fuzz_engine_paths_vs_oracle(engine, case, path):
    n, eu, ev, w, seed, rr = case
    ref = O.c_local_max(n, eu, ev, w, seed, rr)
    eng = engine
    eng.set_algo("auto")
    eng.set_static_order(None)
    if path in ("compact", "scan"):
        eng.set_algo(path)
    if path == "static":
        eng.set_static_order(seed if not rr else None)
    if path == "device" and len(eu):
        import torch
        eng.load_graph_device(n, torch.from_numpy(np.ascontiguousarray(eu)).cuda(),
                              torch.from_numpy(np.ascontiguousarray(ev)).cuda(),
                              torch.from_numpy(np.ascontiguousarray(w)).cuda())
    else:
        eng.load_graph(_graph(n, eu, ev, w))
    eng.set_algo("auto")
    eng.set_static_order(None)
    mate, ids, rounds = eng.match_raw(seed, rr)
    assert np.array_equal(mate, ref.mate)
    assert np.array_equal(ids, ref.matched_ids)
    assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in rounds] == ref.rounds


@settings(max_examples=120, deadline=None, suppress_health_check=list(HealthCheck))
@given(graphs(), st.integers(2, 5), st.sampled_from(["auto", "compact"]))
def test_fuzz_partitioned_vs_oracle(case, p, algo):
    """bsp_local_max's p-invariance (test_bsp.py:68-87): the partitioned
    engine (p partitions emulated on one B200) equals the sequential oracle"""
    from paper_1302_4587_b200.dist import local_max_dist
    n, eu, ev, w, seed, rr = case
    if p > n:
        return
    ref = O.c_local_max(n, eu, ev, w, seed, rr)
    matching, trace = local_max_dist(_graph(n, eu, ev, w), p, seed, rr, algo=algo)
    assert np.array_equal(matching.mate, ref.mate)
    assert np.array_equal(matching.sorted_edge_ids(), ref.matched_ids)
    assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in trace.rounds] == ref.rounds
