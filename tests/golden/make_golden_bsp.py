"""bsp.npz: the UNMODIFIED reference's bsp_local_max RoundMessages
(bsp.py:29-41, :148-199).  Run in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_bsp.py

Per case (generator, size, alpha, seed, p, rerandomize): one row per round
(round_index, candidate_records, bytes_estimate, cut_edges_surviving,
status_records).
"""

from __future__ import annotations

import os

import numpy as np

from locmax import gen_random, gen_rgg
from locmax.bsp import bsp_local_max

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    cases, rows, off = [], [], [0]
    for kind, size, alpha, seed in [("random", 512, 4, 8), ("random", 2000, 3, 1), ("rgg", 11, 0, 4),
                                    ("random", 300, 2, 5)]:
        g = gen_random(size, alpha, seed) if kind == "random" else gen_rgg(size, seed)
        for p in (1, 2, 3, 8):
            for rr in (True, False):
                _, tr = bsp_local_max(g, p, seed, rr)
                cases.append((0 if kind == "random" else 1, size, alpha, seed, p, int(rr)))
                for m in tr.messages:
                    rows.append((m.round_index, m.candidate_records, m.bytes_estimate, m.cut_edges_surviving,
                                 m.status_records))
                off.append(len(rows))
    np.savez_compressed(os.path.join(HERE, "bsp.npz"), cases=np.array(cases, dtype=np.int64),
                        rows=np.array(rows, dtype=np.int64), off=np.array(off, dtype=np.int64))


if __name__ == "__main__":
    main()
