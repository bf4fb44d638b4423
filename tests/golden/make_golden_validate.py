"""validate.npz: the UNMODIFIED reference's validate_matching (graph.py:212-237)
on matchings with each kind of offence.  Run in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_validate.py

Per case: the graph (gen_random(n, alpha, seed)), the matched ids and mate
table handed to validate_matching, and its (valid, maximal) flags.
"""

from __future__ import annotations

import os

import numpy as np

from locmax import gen_random, local_max_seq
from locmax.graph import Matching, validate_matching

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(11)
    rows = {k: [] for k in ("n", "alpha", "seed", "ids_off", "mate_off", "valid", "maximal", "kind")}
    ids_all, mate_all = [], []
    io = mo = 0
    rows["ids_off"].append(0)
    rows["mate_off"].append(0)
    kinds = ["ok", "drop", "disagree", "shared", "stray", "range", "length"]
    for case in range(40):
        n = int(rng.integers(50, 400))
        alpha = int(rng.integers(1, 5))
        seed = int(rng.integers(0, 1000))
        g = gen_random(n, alpha, seed)
        mm, _ = local_max_seq(g, seed)
        ids = sorted(mm.edges)
        mate = np.array(mm.mate)
        kind = kinds[case % len(kinds)]
        e = ids[int(rng.integers(0, len(ids)))] if ids else None
        if kind == "drop" and e is not None:
            ids = [k for k in ids if k != e]
            u, v = g.endpoints(e)
            mate[u] = mate[v] = -1
        elif kind == "disagree" and e is not None:
            mate[g.edge_u[e]] = -1
        elif kind == "shared" and e is not None:
            u = int(g.edge_u[e])
            other = [k for k in range(g.num_edges) if k != e and u in g.endpoints(k)]
            if other:
                ids = sorted(set(ids) | {other[0]})
        elif kind == "stray":
            free = np.nonzero(mate == -1)[0]
            if free.size:
                mate[free[0]] = 0 if free[0] != 0 else 1
        elif kind == "range":
            ids = ids + [g.num_edges + 3]
        elif kind == "length":
            mate = mate[:-1]
        chk = validate_matching(g, Matching(frozenset(ids), mate))
        rows["n"].append(n)
        rows["alpha"].append(alpha)
        rows["seed"].append(seed)
        rows["valid"].append(chk.valid)
        rows["maximal"].append(chk.maximal)
        rows["kind"].append(kinds.index(kind))
        ids_all.extend(ids)
        mate_all.extend(mate.tolist())
        io += len(ids)
        mo += mate.size
        rows["ids_off"].append(io)
        rows["mate_off"].append(mo)
    np.savez_compressed(os.path.join(HERE, "validate.npz"), ids=np.array(ids_all, dtype=np.int64),
                        mate=np.array(mate_all, dtype=np.int64),
                        **{k: np.array(v) for k, v in rows.items()})


if __name__ == "__main__":
    main()
