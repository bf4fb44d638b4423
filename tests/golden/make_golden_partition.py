"""partition.npz: the UNMODIFIED reference's partition_graph (bsp.py:60-98)
on graphs with flat and skewed degrees, for p up to n.  Run in the build
container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_partition.py

Per case: (generator, size, alpha, seed, p) -> bounds, the cut edge count,
degree_imbalance and cut_fraction.
"""

from __future__ import annotations

import os

import numpy as np

from locmax import gen_random, gen_rgg
from locmax.bsp import partition_graph

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rows = []
    bounds = []
    for kind, size, alpha, seed in [("random", 64, 2, 1), ("random", 1000, 3, 2), ("random", 4096, 4, 0),
                                    ("rgg", 10, 0, 3), ("rgg", 12, 0, 4), ("random", 9, 1, 5)]:
        g = gen_random(size, alpha, seed) if kind == "random" else gen_rgg(size, seed)
        for p in (1, 2, 3, 4, 7, 8, 16, g.num_vertices // 2, g.num_vertices):
            if p < 1 or p > g.num_vertices:
                continue
            part = partition_graph(g, p)
            rows.append((0 if kind == "random" else 1, size, alpha, seed, p, int(part.cut_edges.size),
                         float(part.degree_imbalance), float(part.cut_fraction), len(bounds)))
            bounds.extend(part.bounds.tolist())
    r = np.array(rows, dtype=object)
    np.savez_compressed(os.path.join(HERE, "partition.npz"),
                        kind=r[:, 0].astype(np.int64), size=r[:, 1].astype(np.int64), alpha=r[:, 2].astype(np.int64),
                        seed=r[:, 3].astype(np.int64), p=r[:, 4].astype(np.int64), cut=r[:, 5].astype(np.int64),
                        imbalance=r[:, 6].astype(np.float64), cut_fraction=r[:, 7].astype(np.float64),
                        boff=r[:, 8].astype(np.int64), bounds=np.array(bounds, dtype=np.int64))


if __name__ == "__main__":
    main()
