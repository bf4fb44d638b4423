"""Golden fixtures for the red-blue matching (rbm, matchers.py:357-410) from the
UNMODIFIED reference.  Run in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_rbm.py

rbm.npz: for each case (raw graph arrays after the reference's own generator
or build_graph, seed) the reference's sorted matched ids, mate array and
RoundStats trace, plus vertex_coins vectors (tiebreak.py:62-71).
"""

from __future__ import annotations

import os

import numpy as np

from locmax import build_graph, gen_random, gen_rgg
from locmax.generate import with_unit_weights
from locmax.matchers import rbm
from locmax.tiebreak import round_seed, vertex_coins

HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    out = {}
    cases = []
    for n, alpha, s in [(64, 2, 1), (300, 3, 2), (1000, 4, 3), (2000, 2, 4), (500, 8, 5)]:
        cases.append(("random", gen_random(n, alpha, s)))
    for x, s in [(8, 1), (10, 2), (11, 3)]:
        cases.append(("rgg", gen_rgg(x, s)))
    cases.append(("unit", with_unit_weights(gen_random(400, 4, 9))))
    # ties, -0.0 and a few equal weights
    rng = np.random.default_rng(11)
    el = [(int(a), int(b), float(w)) for a, b, w in zip(rng.integers(0, 150, 700), rng.integers(0, 150, 700),
                                                         rng.choice([0.0, -0.0, 0.5, 1.0, 2.0], 700))]
    cases.append(("ties", build_graph(el)))
    for k, (kind, g) in enumerate(cases):
        out[f"c{k}_n"] = np.array([g.num_vertices])
        out[f"c{k}_u"] = np.asarray(g.edge_u, dtype=np.int64)
        out[f"c{k}_v"] = np.asarray(g.edge_v, dtype=np.int64)
        out[f"c{k}_w"] = np.asarray(g.edge_weight, dtype=np.float64)
        for seed in (0, 1, 7):
            m, trace = rbm(g, seed)
            out[f"c{k}_s{seed}_ids"] = m.sorted_edge_ids()
            out[f"c{k}_s{seed}_mate"] = np.asarray(m.mate, dtype=np.int64)
            out[f"c{k}_s{seed}_rounds"] = np.array([[r.edges_before, r.edges_matched, r.edges_removed]
                                                    for r in trace.rounds], dtype=np.int64).reshape(-1, 3)
    out["cases"] = np.array([len(cases)])
    ids = np.arange(0, 5000, 7, dtype=np.int64)
    coins = []
    for s in (0, 1, 2**64 - 1):
        for r in (0, 1, 5):
            rs = round_seed(s, r, True)
            coins.append(vertex_coins(rs, ids))
    out["coin_ids"] = ids
    out["coins"] = np.array(coins)
    np.savez_compressed(os.path.join(HERE, "rbm.npz"), **out)
    print("wrote rbm.npz with", len(cases), "graphs x 3 seeds")


if __name__ == "__main__":
    main()
