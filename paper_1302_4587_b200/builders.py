"""Graph construction on the device: build_graph and synthetic generators.

* :func:`build_graph` -- ``locmax.graph.build_graph`` (graph.py:59-119): same
  signature, validation messages, self-loop removal, parallel-pair collapse
  and first-occurrence edge numbering, computed by ``lmx_build_graph``
  (csrc/lmx_build.cu) on the GPU.
* :func:`gen_rmat` -- RMAT(a, b, c) with ``edge_factor * 2**scale`` raw edges,
  U[0,1) weights, optional Graph500-style relabelling, then build_graph
  semantics (the configs C3 / N★ / C5 of BASELINE.json; the reference has no
  RMAT generator).
"""

from __future__ import annotations

import numpy as np

from .engine import Engine, default_engine
from .graph import Graph


def build_graph(edge_list, num_vertices: int | None = None, device: int = 0) -> Graph:
    """graph.py:59-119 on the device.  ``edge_list``: iterable of (u, v, w)
    triples, or a tuple of three equal-length arrays."""
    if isinstance(edge_list, tuple) and len(edge_list) == 3 and hasattr(edge_list[0], "__len__") \
            and not isinstance(edge_list[0], (int, float)):
        u, v, w = (np.asarray(x) for x in edge_list)
    else:
        triples = list(edge_list)
        if triples:
            u = np.fromiter((int(t[0]) for t in triples), dtype=np.int64, count=len(triples))
            v = np.fromiter((int(t[1]) for t in triples), dtype=np.int64, count=len(triples))
            w = np.fromiter((float(t[2]) for t in triples), dtype=np.float64, count=len(triples))
        else:
            u = v = np.empty(0, dtype=np.int64)
            w = np.empty(0, dtype=np.float64)
    eng = default_engine(device)
    eng.build_graph(u, v, w, num_vertices)
    return eng.export_graph()


def gen_rmat(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19, c: float = 0.19,
             seed: int = 1, permute: bool = True, engine: Engine | None = None,
             export: bool = True) -> Graph | None:
    """Generate (and load into ``engine``) an RMAT graph; optionally export it to host."""
    eng = engine or default_engine(0)
    eng.gen_rmat(scale, edge_factor, a, b, c, seed, permute)
    return eng.export_graph() if export else None


def gen_rgg(x: int, seed: int, weight_mode: str = "euclidean", engine: Engine | None = None,
            export: bool = True) -> Graph | None:
    """``locmax.gen_rgg`` (generate.py:113-143) on the device -- the identical
    graph (points, Morton numbering, edge order, weights).  Loads it into
    ``engine``; optionally exports it to host."""
    eng = engine or default_engine(0)
    eng.gen_rgg(x, seed, weight_mode)
    return eng.export_graph() if export else None
