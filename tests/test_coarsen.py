"""Coarsening pipeline (config C4): mesh generator, ratings, contraction and the
per-level matchings equal the oracle's restatement level by level."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O


def test_oracle_mesh_shape():
    for side in (2, 3, 17):
        n, eu, ev, w = O.mesh_edges(side, 3)
        assert n == side * side and eu.size == (side - 1) * (3 * side - 1)
        assert np.all(eu != ev) and np.all(w == 1.0)
        key = np.minimum(eu, ev) * n + np.maximum(eu, ev)
        assert np.unique(key).size == key.size            # simple graph
        deg = np.bincount(np.concatenate([eu, ev]), minlength=n)
        assert deg.max() <= 8


def test_oracle_contract_conserves_weight():
    n, eu, ev, w = O.mesh_edges(16, 1)
    c = np.ones(n)
    res = O.c_local_max(n, eu, ev, O.ratings(eu, ev, w, c), 1)
    nc, ceu, cev, cw, cc, cid = O.contract(n, eu, ev, w, c, res.mate)
    assert nc == n - res.matched_ids.size
    assert cc.sum() == n
    internal = w[cid[eu] == cid[ev]].sum()
    assert cw.sum() + internal == w.sum()
    assert np.all(ceu < cev)
    assert np.all(np.diff(ceu * nc + cev) > 0)             # ascending, merged


@pytest.mark.gpu
@pytest.mark.parametrize("side", [2, 5, 64])
def test_device_mesh_matches_oracle(engine, side):
    from paper_1302_4587_b200.coarsen import mesh
    n, eu, ev, w = mesh(side, 7, engine)
    on, oeu, oev, ow = O.mesh_edges(side, 7)
    assert n == on
    assert np.array_equal(eu.cpu().numpy(), oeu) and np.array_equal(ev.cpu().numpy(), oev)
    assert np.array_equal(w.cpu().numpy(), ow)


@pytest.mark.gpu
@pytest.mark.parametrize("side,seed", [(32, 0), (64, 3), (128, 5)])
def test_coarsening_levels_match_oracle(engine, side, seed):
    from paper_1302_4587_b200.coarsen import coarsen, mesh
    n, eu, ev, w = mesh(side, seed, engine)
    levels, final = coarsen(n, eu, ev, w, seed=seed, min_n=64, keep_mates=True, engine=engine)
    on, oeu, oev, ow = O.mesh_edges(side, seed)
    ref = O.coarsen_levels(on, oeu, oev, ow, seed=seed, min_n=64)
    assert len(levels) == len(ref) - 1
    for lev, (rn, rm, res) in zip(levels, ref):
        assert (lev.n, lev.m) == (rn, rm)
        assert np.array_equal(lev.mate, res.mate)
        assert lev.matched == res.matched_ids.size
        assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in lev.rounds] == res.rounds
    assert final == (ref[-1][0], ref[-1][1])
