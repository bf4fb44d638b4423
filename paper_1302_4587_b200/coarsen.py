"""Multilevel coarsening by repeated local max matching + contraction (config C4).

This is the paper's motivating application: graph-partitioning coarsening
(``PAPER.md:32-35,342,407-411,474-478``).  The reference ships only the
matching step (``matchers.py:61``) and no contraction (``SPEC.md:16``).  Each
level:

1. ``r(e) = w(e)^2 / (c(u) c(v))``: edge rating from edge weight w and node
   weight c (unit weights at level 0, so every level-0 rating is 1.0).
2. Local max matching on the ratings (``lmx_match``), with seed + level.
3. Contraction (``lmx_contract``):
   * a matched pair or an unmatched vertex becomes one coarse vertex,
     numbered by its smaller member in ascending order;
   * node weights add;
   * parallel edges merge by summing w, listed in ascending (min, max)
     coarse-pair order.

Coarsening stops when the coarse graph has fewer than ``min_n`` vertices or
shrank by less than ``min_shrink``.  Everything stays on the device; only
per-level scalars come back.  ``oracle/oracle.py:coarsen_levels`` restates
the pipeline for the parity tests.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from .engine import LMX_OK, Engine, _raise, default_engine


@dataclass
class Level:
    n: int
    m: int
    matched: int = 0
    rounds: list = field(default_factory=list)
    mate: np.ndarray | None = None        # host copy when keep_mates=True
    match_ms: float = 0.0                 # device round loop of this level
    stage_ms: dict = field(default_factory=dict)   # profile=True: synchronised stage times


def _bind(lib):
    if getattr(lib, "_coarsen_bound", False):
        return
    p, i64, u64, c_int = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
    lib.lmx_mesh_edges.restype = c_int
    lib.lmx_mesh_edges.argtypes = [p, i64, u64, p, p, p, ctypes.POINTER(i64)]
    lib.lmx_ratings.restype = c_int
    lib.lmx_ratings.argtypes = [p, i64, p, p, p, p, p]
    lib.lmx_contract.restype = c_int
    lib.lmx_contract.argtypes = [p, i64, i64, p, p, p, p, p, p, ctypes.POINTER(i64), ctypes.POINTER(i64),
                                 p, p, p, p]
    lib._coarsen_bound = True


def _chk(eng, rc, what):
    if rc != LMX_OK:
        _raise(rc, f"{what}: " + eng._lib.lmx_last_error(eng._h).decode())


def mesh(side: int, seed: int = 0, engine: Engine | None = None):
    """side x side jittered-grid triangulation on the device: (n, eu, ev, w) CUDA tensors."""
    import torch
    eng = engine or default_engine(0)
    _bind(eng._lib)
    m_cap = (side - 1) * (3 * side - 1)
    eu = torch.empty(m_cap, dtype=torch.int64, device="cuda")
    ev = torch.empty(m_cap, dtype=torch.int64, device="cuda")
    w = torch.empty(m_cap, dtype=torch.float64, device="cuda")
    m = ctypes.c_int64()
    _chk(eng, eng._lib.lmx_mesh_edges(eng._h, side, seed, eu.data_ptr(), ev.data_ptr(), w.data_ptr(),
                                      ctypes.byref(m)), "lmx_mesh_edges")
    return side * side, eu[: m.value], ev[: m.value], w[: m.value]


def coarsen(n: int, eu, ev, w, seed: int = 0, min_n: int = 1024, min_shrink: float = 0.05,
            max_levels: int = 64, keep_mates: bool = False, engine: Engine | None = None,
            profile: bool = False):
    """Coarsen the device graph (eu, ev int64 / w float64 CUDA tensors).

    Returns ``(levels, (n_coarse, m_coarse))``.  ``levels[i]`` describes the
    matching of level i; the last contraction's result is the coarsest graph.
    """
    import torch
    eng = engine or default_engine(0)
    _bind(eng._lib)
    lib = eng._lib
    dev = eu.device
    c = torch.ones(n, dtype=torch.float64, device=dev)
    c0 = torch.empty(max(n, 1), dtype=torch.float64, device=dev)   # node weights, ping-pong with buf["cc"]
    levels = []
    marks = {}

    def mark(name):
        if profile:
            torch.cuda.synchronize()
            marks[name] = time.perf_counter()

    # Level-0-sized buffers, reused by every level (coarse graphs only shrink):
    # one allocation set per call instead of one per level
    m0, n0 = int(eu.numel()), n
    buf = {k: torch.empty(max(sz, 1), dtype=dt, device=dev) for k, sz, dt in (
        ("r", m0, torch.float64), ("mate", n0, torch.int64), ("ids", n0 // 2 + 1, torch.int64),
        ("cid", n0, torch.int64), ("cc", n0, torch.float64))}
    side = [{k: torch.empty(max(m0, 1), dtype=dt, device=dev) for k, dt in
             (("eu", torch.int64), ("ev", torch.int64), ("w", torch.float64))} for _ in range(2)]
    torch.cuda.synchronize(dev)   # the buffers above come from torch's stream; the engine runs on its own
    for lvl in range(max_levels):
        mark("start")
        m = int(eu.numel())
        r = buf["r"][:m]
        _chk(eng, lib.lmx_ratings(eng._h, m, eu.data_ptr(), ev.data_ptr(), w.data_ptr(), c.data_ptr(),
                                  r.data_ptr()), "lmx_ratings")
        mark("ratings")
        eng.load_graph_device(n, eu, ev, r)
        mark("load")
        mate = buf["mate"][: max(n, 1)]
        ids = buf["ids"][: max(n // 2 + 1, 1)]
        matched = eng.match_device(seed + lvl, mate, ids)
        mark("match")
        lev = Level(n, m, matched, eng.last_rounds(), match_ms=eng.last_timing()["rounds_ms"])
        if keep_mates:
            lev.mate = mate[:n].cpu().numpy()
        levels.append(lev)
        out = side[lvl & 1]
        cid = buf["cid"][: max(n, 1)]
        ceu, cev, cw = out["eu"], out["ev"], out["w"]
        cc = (buf["cc"] if lvl % 2 == 0 else c0)[: max(n, 1)]
        nc = ctypes.c_int64()
        mc = ctypes.c_int64()
        _chk(eng, lib.lmx_contract(eng._h, n, m, eu.data_ptr(), ev.data_ptr(), w.data_ptr(), c.data_ptr(),
                                   mate.data_ptr(), cid.data_ptr(), ctypes.byref(nc), ctypes.byref(mc),
                                   ceu.data_ptr(), cev.data_ptr(), cw.data_ptr(), cc.data_ptr()), "lmx_contract")
        mark("contract")
        if profile:
            names = ["start", "ratings", "load", "match", "contract"]
            lev.stage_ms = {b: (marks[b] - marks[a]) * 1e3 for a, b in zip(names, names[1:])}
            lev.stage_ms["algo"] = {"scan": 1.0, "compact": 0.0}[eng.algo()]
        shrink_ok = (n - nc.value) >= min_shrink * n
        n, eu, ev, w, c = nc.value, ceu[: mc.value], cev[: mc.value], cw[: mc.value], cc[: nc.value]
        if n < min_n or not shrink_ok:
            break
    return levels, (n, int(eu.numel()))


def coarsen_mesh(side: int = 4096, seed: int = 0, **kw):
    """Config C4: coarsen the side x side mesh (2^24 vertices at side 4096)."""
    # the process-wide engine (as local_max_b200 uses): its device block cache
    # serves every level's buffers after the first call
    eng = kw.pop("engine", None) or default_engine(0)
    t0 = time.perf_counter()
    n, eu, ev, w = mesh(side, seed, eng)
    levels, final = coarsen(n, eu, ev, w, seed=seed, engine=eng, **kw)
    return levels, final, (time.perf_counter() - t0) * 1000.0
