"""GPU red-blue matching against the reference's rbm
outputs (tests/golden/rbm.npz) and the pinned oracle restatement."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from test_oracle_rbm import GOLD, rbm_cases

pytestmark = pytest.mark.gpu


def _graph(n, eu, ev, w):
    from paper_1302_4587_b200 import Graph
    return Graph(n, eu, ev, w)


@pytest.mark.parametrize("layout", ["auto", "distinct", "general"])
def test_rbm_golden_bit_exact(engine, layout):
    z = np.load(GOLD)
    engine.set_layout(layout)
    try:
        for k, seed, (n, eu, ev, w), ids, mate, rounds in rbm_cases(z):
            if layout == "distinct" and np.unique(w).size < 0.9 * w.size:
                continue   # too many ties for the distinct layout
            g = _graph(n, eu, ev, w)
            engine.load_graph(g)
            m, trace = engine.rbm(g, seed)
            assert np.array_equal(m.sorted_edge_ids(), ids), (k, seed)
            assert np.array_equal(np.asarray(m.mate), mate), (k, seed)
            assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in trace.rounds] == rounds, (k, seed)
    finally:
        engine.set_layout("auto")


@pytest.mark.parametrize("seed", [3, 11])
def test_rbm_random_and_relabelled_rmat_vs_oracle(engine, seed):
    from paper_1302_4587_b200 import run_matcher
    n, eu, ev, w = O.gen_random(20000, 5, seed)
    g = _graph(n, eu, ev, w)
    m, trace = run_matcher(g, "rbm", seed, engine="b200")
    res = O.numpy_rbm(n, eu, ev, w, seed)
    assert np.array_equal(np.asarray(m.mate), res.mate)
    assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in trace.rounds] == res.rounds
    # skewed graph: degree relabelling on; coins use the caller's ids
    engine.gen_rmat(12, 8, 0.57, 0.19, 0.19, seed=seed, permute=True)
    assert engine.relabeled()
    gr = engine.export_graph()
    m, trace = engine.rbm(gr, seed)
    res = O.numpy_rbm(gr.num_vertices, gr.edge_u, gr.edge_v, gr.edge_weight, seed)
    assert np.array_equal(np.asarray(m.mate), res.mate)
    assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in trace.rounds] == res.rounds
    chk, _ = engine.validate(m)
    assert chk.valid and chk.maximal


def test_rbm_round_limit_raises(engine):
    from paper_1302_4587_b200 import RbmDidNotConverge
    n, eu, ev, w = O.gen_random(2000, 4, 1)
    g = _graph(n, eu, ev, w)
    engine.load_graph(g)
    with pytest.raises(RbmDidNotConverge):
        engine.rbm(g, 1, max_rounds=1)
