"""The PRAM entry point (pram_local_max, pram.py:276-315): same matching as the
sequential loop and the same ``trace.slot_ops`` linear-work meter, pinned
against the reference's own values (tests/golden/pram.npz, made by
tests/golden/make_golden_pram.py)."""

from __future__ import annotations

import hashlib
import os

import numpy as np
import pytest

from conftest import small_cases, small_runs

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "pram.npz")


def _digest(mate) -> str:
    return hashlib.sha256(np.ascontiguousarray(mate, dtype=np.int64).tobytes()).hexdigest()[:16]


def _cases(golden_small):
    z = np.load(GOLD)
    graphs = {gi: (n, built) for gi, n, _, built, _ in small_cases(golden_small)}
    runs = {(gi, seed, rr): rounds for gi, seed, rr, _, _, rounds in small_runs(golden_small)}
    for k in range(len(z["graph"])):
        gi, seed, rr = int(z["graph"][k]), int(z["seed"][k]), bool(z["rr"][k])
        yield graphs[gi], seed, rr, int(z["slot_ops"][k]), int(z["rounds"][k]), str(z["mate_digest"][k]), \
            runs.get((gi, seed, rr))


def test_slot_ops_formula_matches_reference(golden_small):
    """slot_ops = n + 3m + 3 * sum(m_r), checked on the reference's own meter."""
    done = 0
    for (n, (eu, ev, w)), seed, rr, slot_ops, n_rounds, _, rounds in _cases(golden_small):
        if rounds is None:
            continue
        assert len(rounds) == n_rounds
        assert n + 3 * len(eu) + 3 * sum(r[0] for r in rounds) == slot_ops
        done += 1
    assert done > 20


@pytest.mark.gpu
def test_pram_entry_matches_reference(golden_small):
    from paper_1302_4587_b200 import Graph, pram_local_max_b200
    done = 0
    for (n, (eu, ev, w)), seed, rr, slot_ops, n_rounds, digest, _ in _cases(golden_small):
        matching, trace = pram_local_max_b200(Graph(n, eu, ev, w), seed, checked=bool(done % 2), rerandomize=rr)
        assert trace.slot_ops == slot_ops
        assert len(trace.rounds) == n_rounds
        assert _digest(matching.mate) == digest
        done += 1
    assert done > 100


@pytest.mark.gpu
def test_run_matcher_pram_engine():
    from oracle import oracle as O
    from paper_1302_4587_b200 import Graph, run_matcher
    n, eu, ev, w = O.gen_random(1 << 10, 4, 2)
    g = Graph(n, eu, ev, w)
    a, _ = run_matcher(g, "localmax", 2, engine="b200")
    b, tb = run_matcher(g, "localmax", 2, engine="b200-pram")
    assert a == b and tb.slot_ops > 0


@pytest.mark.gpu
def test_pram_cross_pointers_and_write_log():
    """lmx_pram_cross: the reference incidence layout's cross pointers
    (pram.py:127-166) -- each slot points at the other slot of its edge, an
    involution -- built with 4 exclusive-write steps of m writes each."""
    from oracle import oracle as O
    from paper_1302_4587_b200 import Engine, Graph
    for n, eu, ev, w in (O.gen_random(500, 3, 1), O.gen_rgg(10, 2), O.gen_random(64, 2, 4, unit=True)):
        g = Graph(n, eu, ev, w)
        with Engine(0) as eng:
            eng.load_graph(g)
            log, cross = eng.pram_cross(want_cross=True)
        m = len(eu)
        # graph.py:108-115 layout, numpy: slots sorted by (vertex, edge id)
        sv = np.concatenate([eu, ev])
        se = np.concatenate([np.arange(m), np.arange(m)])
        order = np.lexsort((se, sv))
        sv, se = sv[order], se[order]
        idx = np.arange(2 * m)
        want = np.empty(2 * m, dtype=np.int64)
        pos = {}
        for i, e in zip(idx.tolist(), se.tolist()):
            pos.setdefault(e, []).append(i)
        for e, (a, b) in pos.items():
            want[a], want[b] = b, a
        assert np.array_equal(cross, want)
        assert log == {"steps": 4, "writes": 4 * m, "conflicts": 0, "bad_slot": -1}


@pytest.mark.gpu
def test_reference_pram_assertions_with_b200_engine():
    """test_pram.py:164-184 with pram_local_max replaced by the B200 engine:
    equal matching, equal round count, a write log without conflicts; and
    the rerandomize flag respected."""
    from oracle import oracle as O
    from paper_1302_4587_b200 import Graph, local_max_b200, pram_local_max_b200
    cases = [(O.gen_rgg(12, 7), 7), (O.gen_random(512, 4, 3), 3), (O.gen_random(512, 16, 4), 11),
             ((2, np.array([0]), np.array([1]), np.array([1.0])), 0)]
    for (n, eu, ev, w), seed in cases:
        g = Graph(n, eu, ev, w)
        ref = O.c_local_max(n, eu, ev, w, seed, True)
        par_matching, par_trace = pram_local_max_b200(g, seed, checked=True)
        assert np.array_equal(np.asarray(par_matching.mate), ref.mate)
        assert par_trace.total_rounds == len(ref.rounds)
        assert par_trace.write_log.conflicts == 0
    n, eu, ev, w = O.gen_rgg(10, 2)
    g = Graph(n, eu, ev, w)
    for flag in (True, False):
        a, _ = local_max_b200(g, 5, rerandomize=flag)
        b, _ = pram_local_max_b200(g, 5, rerandomize=flag)
        assert a == b
