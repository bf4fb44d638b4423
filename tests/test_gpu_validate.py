"""GPU validate_matching and Matching.weight against the
CPU statement of graph.py:212-237 and numpy's edge_weight[ids].sum()."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _graph(n, eu, ev, w):
    from paper_1302_4587_b200 import Graph
    return Graph(n, eu, ev, w)


def _ref_weight(g, ids):
    # graph.py:54-56: float(edge_weight[sorted ids].sum())
    return float(np.asarray(g.edge_weight)[np.sort(ids)].sum()) if len(ids) else 0.0


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("kind", ["random", "rgg", "unit"])
def test_validate_matches_cpu_and_weight_bit_exact(engine, seed, kind):
    from paper_1302_4587_b200 import validate_matching
    if kind == "rgg":
        n, eu, ev, w = O.gen_rgg(12, seed)
    else:
        n, eu, ev, w = O.gen_random(5000, 6, seed, unit=(kind == "unit"))
    g = _graph(n, eu, ev, w)
    engine.load_graph(g)
    m, _ = engine.match(g, seed, True)
    chk, weight = engine.validate(m)
    ref = validate_matching(g, m)
    assert (chk.valid, chk.maximal) == (ref.valid, ref.maximal) == (True, True)
    assert weight == _ref_weight(g, m.sorted_edge_ids())   # bit-identical, not approximately


def test_validate_detects_each_offence(engine):
    from paper_1302_4587_b200 import Matching, validate_matching
    n, eu, ev, w = O.gen_random(3000, 5, 7)
    g = _graph(n, eu, ev, w)
    engine.load_graph(g)
    m, _ = engine.match(g, 7, True)
    ids = m.sorted_edge_ids()
    mate = np.array(m.mate)

    def both(ids_, mate_):
        mm = Matching(np.asarray(ids_, dtype=np.int64), np.asarray(mate_, dtype=np.int64))
        got, _ = engine.validate(mm)
        ref = validate_matching(g, mm)
        return got, ref

    # a matched edge dropped (mate made consistent): valid, not maximal
    e = int(ids[0])
    mate2 = mate.copy()
    mate2[eu[e]] = -1
    mate2[ev[e]] = -1
    got, ref = both(ids[1:], mate2)
    assert (got.valid, got.maximal) == (ref.valid, ref.maximal) == (True, False)
    # mate table disagrees with a matched edge
    mate3 = mate.copy()
    mate3[eu[e]] = -1
    got, ref = both(ids, mate3)
    assert (got.valid, got.maximal) == (ref.valid, ref.maximal) == (False, False)
    assert "disagrees" in got.detail
    # a vertex shared by two matched edges
    u = int(eu[e])
    other = [k for k in range(len(eu)) if k != e and (eu[k] == u or ev[k] == u)]
    if other:
        got, ref = both(np.sort(np.append(ids, other[0])), mate)
        assert (got.valid, got.maximal) == (ref.valid, ref.maximal) == (False, False)
    # a stray mate entry
    free = np.nonzero(mate == -1)[0]
    if free.size:
        mate4 = mate.copy()
        mate4[free[0]] = 0
        got, ref = both(ids, mate4)
        assert (got.valid, got.maximal) == (ref.valid, ref.maximal) == (False, False)
    # an edge id out of range
    got, _ = both(np.append(ids, len(eu) + 5), mate)
    assert not got.valid and "out of range" in got.detail
    # wrong mate length
    got, ref = both(ids, mate[:-1])
    assert (got.valid, got.maximal) == (ref.valid, ref.maximal) == (False, False)


def test_validate_empty_matching_and_rmat(engine):
    from paper_1302_4587_b200 import Matching
    n, eu, ev, w = O.gen_random(500, 3, 2)
    g = _graph(n, eu, ev, w)
    engine.load_graph(g)
    empty = Matching(np.zeros(0, dtype=np.int64), np.full(n, -1, dtype=np.int64))
    chk, weight = engine.validate(empty)
    assert chk.valid and not chk.maximal and weight == 0.0
    # device-built RMAT: the weight of a large matching, bit-exact
    engine.gen_rmat(16, 16, 0.57, 0.19, 0.19, seed=3, permute=True)
    gr = engine.export_graph()
    m, _ = engine.match(gr, 5, True)
    chk, weight = engine.validate(m)
    assert chk.valid and chk.maximal
    assert weight == _ref_weight(gr, m.sorted_edge_ids())
