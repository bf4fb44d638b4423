"""The oracle's red-blue matching restatement pinned against the reference's
own rbm (matchers.py:357-410) and vertex_coins (tiebreak.py:62-71) outputs
(tests/golden/rbm.npz, made by tests/golden/make_golden_rbm.py)."""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "rbm.npz")


@pytest.fixture(scope="module")
def rbm_gold():
    return np.load(GOLD)


def rbm_cases(z):
    for k in range(int(z["cases"][0])):
        g = (int(z[f"c{k}_n"][0]), z[f"c{k}_u"], z[f"c{k}_v"], z[f"c{k}_w"])
        for seed in (0, 1, 7):
            p = f"c{k}_s{seed}_"
            yield k, seed, g, z[p + "ids"], z[p + "mate"], [tuple(int(x) for x in r) for r in z[p + "rounds"]]


def test_vertex_coins_match_reference(rbm_gold):
    ids = rbm_gold["coin_ids"]
    i = 0
    for s in (0, 1, 2**64 - 1):
        for r in (0, 1, 5):
            assert np.array_equal(O.vertex_coins(O.round_seed(s, r, True), ids), rbm_gold["coins"][i])
            i += 1


def test_numpy_rbm_matches_reference(rbm_gold):
    for k, seed, (n, eu, ev, w), ids, mate, rounds in rbm_cases(rbm_gold):
        res = O.numpy_rbm(n, eu, ev, w, seed)
        assert np.array_equal(res.matched_ids, ids), (k, seed)
        assert np.array_equal(res.mate, mate), (k, seed)
        assert res.rounds == rounds, (k, seed)
