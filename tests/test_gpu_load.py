"""Loading from host memory (lmx_load_graph, where=LMX_HOST): the endpoint
arrays are narrowed and range-checked by host threads into a pinned staging
ring (lmx_setup.cu load_host_narrowed).  The loaded graph must not depend on
the path (pageable / page-locked inputs, thread count, device-resident
inputs), and a bad edge must be reported by its first index, as the reference's
Graph construction does (graph.py:70-90)."""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _graph(n, eu, ev, w):
    from paper_1302_4587_b200 import Graph
    return Graph(n, eu, ev, w)


def _pinned(a):
    import torch
    t = torch.empty(a.shape[0], dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    out = t.numpy()
    out[:] = a
    return out, t


def _run(engine, g, seed=5):
    engine.load_graph(g)
    mate, ids, rounds = engine.match_raw(seed, True)
    return mate.copy(), ids.copy(), list(rounds)


@pytest.mark.parametrize("threads", [None, "1", "3"])
def test_host_paths_identical(engine, threads, monkeypatch):
    if threads:
        monkeypatch.setenv("LMX_LOAD_THREADS", threads)
    n, eu, ev, w = O.gen_random(200_000, 12, 3)           # 2.4 M edges: many staging blocks
    ref = O.c_local_max(n, eu, ev, w, 5, True)
    got = _run(engine, _graph(n, eu, ev, w))               # pageable arrays
    assert np.array_equal(got[0], ref.mate) and np.array_equal(got[1], ref.matched_ids)
    pu, _tu = _pinned(eu)
    pv, _tv = _pinned(ev)
    pw, _tw = _pinned(w)
    got_p = _run(engine, _graph(n, pu, pv, pw))            # page-locked arrays (weights copied directly)
    assert np.array_equal(got_p[0], got[0]) and np.array_equal(got_p[1], got[1]) and got_p[2] == got[2]


def test_host_load_matches_device_load(engine):
    import torch
    n, eu, ev, w = O.gen_random(100_000, 8, 4)
    host = _run(engine, _graph(n, eu, ev, w))
    du = torch.from_numpy(eu).cuda()
    dv = torch.from_numpy(ev).cuda()
    dw = torch.from_numpy(w).cuda()
    engine.load_graph_device(n, du, dv, dw)
    mate, ids, rounds = engine.match_raw(5, True)
    assert np.array_equal(mate, host[0]) and np.array_equal(ids, host[1])
    assert list(rounds) == host[2]


@pytest.mark.parametrize("pinned", [False, True])
def test_first_bad_edge_reported(engine, pinned, monkeypatch):
    monkeypatch.setenv("LMX_LOAD_THREADS", "4")
    n, eu, ev, w = O.gen_random(100_000, 8, 6)
    m = len(eu)
    keep = []

    def graph(u, v, x):   # fresh arrays per Graph (Graph freezes what it is given)
        arrays = []
        for a in (u, v, x):
            if pinned:
                p, t = _pinned(a)
                keep.append(t)
                arrays.append(p)
            else:
                arrays.append(a.copy())
        return _graph(n, *arrays)

    eu = eu.copy()
    ev = ev.copy()
    late, early = m - 3, m // 2 + 17                      # in different staging blocks
    ev[late] = n + 5                                      # out of range
    good_u = eu[early]
    eu[early] = ev[early]                                 # self-loop, the first bad edge
    with pytest.raises(ValueError, match=f"edge {early}: self-loop"):
        engine.load_graph(graph(eu, ev, w))
    eu[early] = good_u
    with pytest.raises(ValueError, match=f"edge {late}: vertex id out of range"):
        engine.load_graph(graph(eu, ev, w))
    eu2 = eu.copy()
    eu2[7] = -1                                           # negative id: nothing may touch deg[-1]
    with pytest.raises(ValueError, match="edge 7: vertex id out of range"):
        engine.load_graph(graph(eu2, ev, w))
    w2 = w.copy()
    w2[5] = -1.0
    with pytest.raises(ValueError, match="edge 5: weight"):
        engine.load_graph(graph(eu, ev, w2))
    # the engine is usable after the failed loads (the staging ring is idle)
    n2, eu2, ev2, w3 = O.gen_random(50_000, 6, 7)
    ref = O.c_local_max(n2, eu2, ev2, w3, 5, True)
    got = _run(engine, _graph(n2, eu2, ev2, w3))
    assert np.array_equal(got[0], ref.mate) and np.array_equal(got[1], ref.matched_ids)


def test_load_sizes_reuse_ring(engine):
    # small after large after small: the ring is sized by the largest load
    for size in (1_000, 300_000, 10, 40_000):
        n, eu, ev, w = O.gen_random(size, 4, size)
        ref = O.c_local_max(n, eu, ev, w, 5, True)
        got = _run(engine, _graph(n, eu, ev, w))
        assert np.array_equal(got[0], ref.mate) and np.array_equal(got[1], ref.matched_ids)
