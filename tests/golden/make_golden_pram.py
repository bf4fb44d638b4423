"""Golden fixtures for the PRAM entry point (pram_local_max, pram.py:276-315)
from the UNMODIFIED reference.  Run in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_pram.py

pram.npz: for a spread of the small.npz graphs, seeds and rerandomize modes,
the reference's trace.slot_ops (its linear-work meter), the mate array's
digest and the round count.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

from locmax.graph import Graph as RefGraph
from locmax.pram import pram_local_max

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from conftest import small_cases  # noqa: E402


def ref_graph(n, eu, ev, w):
    from locmax import build_graph
    edges = [(int(a), int(b), float(c)) for a, b, c in zip(eu, ev, w)]
    return build_graph(edges, num_vertices=n)


def main() -> None:
    z = np.load(os.path.join(HERE, "small.npz"))
    rows = []
    for gi, n, _, (eu, ev, w), _ in small_cases(z):
        if gi % 5:
            continue
        g = ref_graph(n, eu, ev, w)
        assert isinstance(g, RefGraph) and g.num_edges == len(eu)
        for seed, rr in ((0, True), (3, False), (11, True)):
            matching, trace = pram_local_max(g, seed, rerandomize=rr)
            digest = hashlib.sha256(np.ascontiguousarray(matching.mate, dtype=np.int64).tobytes()).hexdigest()[:16]
            rows.append((gi, seed, int(rr), int(trace.slot_ops), len(trace.rounds), digest))
    out = {
        "graph": np.array([r[0] for r in rows], dtype=np.int64),
        "seed": np.array([r[1] for r in rows], dtype=np.int64),
        "rr": np.array([r[2] for r in rows], dtype=np.int64),
        "slot_ops": np.array([r[3] for r in rows], dtype=np.int64),
        "rounds": np.array([r[4] for r in rows], dtype=np.int64),
        "mate_digest": np.array([r[5] for r in rows]),
    }
    np.savez_compressed(os.path.join(HERE, "pram.npz"), **out)
    print(f"{len(rows)} runs")


if __name__ == "__main__":
    main()
