"""CPU oracle for the local max matching path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and only
as the checker / the timed CPU baseline.  The product package
(``paper_1302_4587_b200``) never imports it.

Contents
--------
* ``c_local_max``     -- ctypes front end of ``lmx_oracle.c`` (restates
  ``matchers.py:61-122``); fast enough for every config up to RMAT-24.
* ``numpy_local_max`` -- a numpy restatement of ``local_max_seq`` that uses
  the same whole-array numpy operations as the reference
  (``np.maximum.at`` scatter-max stages, ``matchers.py:87-119``), so timing it
  times the reference's algorithm at the reference's speed (1 core).
* ``mix64`` / ``round_seed`` / ``edge_salts`` / ``weight_bits`` -- numpy
  restatements of ``tiebreak.py:28-59,105-113``.
* ``gen_random`` / ``gen_rgg`` / ``with_unit_weights`` / ``build_graph_loop``
  -- restatements of ``generate.py:48-143,146-197,219-222`` and
  ``graph.py:59-119`` used to regenerate the reference's instances in tests
  (the reference itself is absent on the GPU box).

Parity pin: ``tests/test_oracle_golden.py`` checks all of the above against
``tests/golden/*.npz``, produced from the unmodified reference by
``tests/golden/make_golden.py``.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liblmx_oracle.so")
_UINT64_MASK = (1 << 64) - 1

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_MIX_A = np.uint64(0xBF58476D1CE4E5B9)
_MIX_B = np.uint64(0x94D049BB133111EB)


def build() -> str:
    """Compile lmx_oracle.c with plain gcc (oracle/Makefile)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "lmx_oracle.c"))
        ):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.lmxo_mix64.restype = ctypes.c_uint64
        lib.lmxo_mix64.argtypes = [ctypes.c_uint64]
        lib.lmxo_round_seed.restype = ctypes.c_uint64
        lib.lmxo_round_seed.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int]
        lib.lmxo_local_max.restype = ctypes.c_int
        p = ctypes.c_void_p
        lib.lmxo_local_max.argtypes = [
            ctypes.c_int64, ctypes.c_int64, p, p, p, ctypes.c_uint64, ctypes.c_int,
            p, p, p, p, ctypes.c_int,
        ]
        lib.lmxo_edge_salts.restype = None
        lib.lmxo_edge_salts.argtypes = [ctypes.c_uint64, p, ctypes.c_int64, p]
        lib.lmxo_rmat_raw.restype = None
        lib.lmxo_rmat_raw.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint32,
                                      ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, p, p, p]
        lib.lmxo_build_graph.restype = ctypes.c_int64
        lib.lmxo_build_graph.argtypes = [ctypes.c_int64, p, p, p, ctypes.c_int64, p, p, p, p]
        _lib = lib
    return _lib


# ---------------------------------------------------------------- tiebreak.py

def mix64(values: np.ndarray) -> np.ndarray:
    """tiebreak.py:28-37."""
    with np.errstate(over="ignore"):
        x = np.asarray(values, dtype=np.uint64) + _GOLDEN
        x ^= x >> np.uint64(30)
        x *= _MIX_A
        x ^= x >> np.uint64(27)
        x *= _MIX_B
        x ^= x >> np.uint64(31)
    return x


def round_seed(seed: int, round_index: int, rerandomize: bool = True) -> int:
    """tiebreak.py:40-52."""
    if round_index < 0:
        raise ValueError("round_index must be nonnegative")
    r = round_index if rerandomize else 0
    base = np.array([seed & _UINT64_MASK], dtype=np.uint64)
    return int(mix64(mix64(base) ^ np.uint64(r))[0])


def edge_salts(round_seed_value: int, edge_ids) -> np.ndarray:
    """tiebreak.py:55-59."""
    ids = np.asarray(edge_ids, dtype=np.uint64)
    return mix64(ids ^ np.uint64(round_seed_value & _UINT64_MASK))


def weight_bits(weights) -> np.ndarray:
    """tiebreak.py:105-113."""
    w = np.asarray(weights, dtype=np.float64) + 0.0
    return w.view(np.uint64)


# ---------------------------------------------------------------- results

@dataclass
class OracleResult:
    mate: np.ndarray          # int64[n], -1 unmatched
    matched_ids: np.ndarray   # int64, ascending
    rounds: list              # [(edges_before, edges_matched, edges_removed)]


def c_local_max(n: int, edge_u, edge_v, edge_weight, seed: int,
                rerandomize: bool = True) -> OracleResult:
    """lmx_oracle.c restatement of matchers.py:61-122."""
    lib = _load()
    eu = np.ascontiguousarray(edge_u, dtype=np.int64)
    ev = np.ascontiguousarray(edge_v, dtype=np.int64)
    w = np.ascontiguousarray(edge_weight, dtype=np.float64)
    m = int(eu.size)
    mate = np.empty(max(n, 1), dtype=np.int64)
    ids = np.empty(max(n // 2 + 1, 1), dtype=np.int64)
    nm = np.zeros(1, dtype=np.int64)
    # a path with monotone weights needs n/2 rounds: retry with room for that
    for max_rounds in (4096, max(4096, n // 2 + 2)):
        rounds = np.zeros(3 * max_rounds, dtype=np.int64)
        r = lib.lmxo_local_max(
            n, m, eu.ctypes.data, ev.ctypes.data, w.ctypes.data,
            seed & _UINT64_MASK, 1 if rerandomize else 0,
            mate.ctypes.data, ids.ctypes.data, nm.ctypes.data, rounds.ctypes.data, max_rounds,
        )
        if r != -2:
            break
    if r < 0:
        raise RuntimeError(f"oracle failed with status {r}")
    rr = rounds[: 3 * r].reshape(r, 3)
    return OracleResult(mate[:n].copy(), ids[: int(nm[0])].copy(),
                        [tuple(int(x) for x in row) for row in rr])


def c_mix64(v: int) -> int:
    return int(_load().lmxo_mix64(v & _UINT64_MASK))


def c_round_seed(seed: int, r: int, rerandomize: bool = True) -> int:
    return int(_load().lmxo_round_seed(seed & _UINT64_MASK, r, 1 if rerandomize else 0))


def c_edge_salts(rs: int, ids) -> np.ndarray:
    a = np.ascontiguousarray(ids, dtype=np.uint64)
    out = np.empty_like(a)
    _load().lmxo_edge_salts(rs & _UINT64_MASK, a.ctypes.data, a.size, out.ctypes.data)
    return out


def numpy_local_max(n: int, edge_u, edge_v, edge_weight, seed: int,
                    rerandomize: bool = True) -> OracleResult:
    """numpy restatement of local_max_seq (matchers.py:61-122), same ops."""
    edge_u = np.asarray(edge_u, dtype=np.int64)
    edge_v = np.asarray(edge_v, dtype=np.int64)
    edge_weight = np.asarray(edge_weight, dtype=np.float64)
    m = edge_u.size
    cand_w = np.zeros(n, dtype=np.uint64)
    cand_s = np.zeros(n, dtype=np.uint64)
    cand_id = np.full(n, -1, dtype=np.int64)
    vertex_matched = np.zeros(n, dtype=bool)
    live = np.arange(m, dtype=np.int64)
    parts = []
    rounds = []
    r = 0
    while live.size:
        rs = round_seed(seed, r, rerandomize)
        wbits = weight_bits(edge_weight[live])
        salts = edge_salts(rs, live)
        us = edge_u[live]
        vs = edge_v[live]
        np.maximum.at(cand_w, us, wbits)
        np.maximum.at(cand_w, vs, wbits)
        tie_u = cand_w[us] == wbits
        tie_v = cand_w[vs] == wbits
        np.maximum.at(cand_s, us[tie_u], salts[tie_u])
        np.maximum.at(cand_s, vs[tie_v], salts[tie_v])
        tie_u &= cand_s[us] == salts
        tie_v &= cand_s[vs] == salts
        np.maximum.at(cand_id, us[tie_u], live[tie_u])
        np.maximum.at(cand_id, vs[tie_v], live[tie_v])
        won = (cand_id[us] == live) & (cand_id[vs] == live)
        new_edges = live[won]
        parts.append(new_edges)
        vertex_matched[us[won]] = True
        vertex_matched[vs[won]] = True
        alive = ~(vertex_matched[us] | vertex_matched[vs])
        for ends in (us[alive], vs[alive]):
            cand_w[ends] = 0
            cand_s[ends] = 0
            cand_id[ends] = -1
        survivors = live[alive]
        rounds.append((int(live.size), int(new_edges.size), int(live.size - survivors.size)))
        live = survivors
        r += 1
    matched = np.sort(np.concatenate(parts)) if parts else np.empty(0, dtype=np.int64)
    mate = np.full(n, -1, dtype=np.int64)
    if matched.size:
        mate[edge_u[matched]] = edge_v[matched]
        mate[edge_v[matched]] = edge_u[matched]
    return OracleResult(mate, matched, rounds)


# ---------------------------------------------------------------- red-blue matching
_COIN_STREAM = np.uint64(0xD6E8FEB86659FD93)   # tiebreak.py:25


def vertex_coins(round_seed_value: int, vertex_ids) -> np.ndarray:
    """tiebreak.py:62-71: True = blue; a stream separate from the edge salts."""
    ids = np.asarray(vertex_ids, dtype=np.uint64)
    h = mix64(ids ^ np.uint64(round_seed_value & _UINT64_MASK) ^ _COIN_STREAM)
    return (h & np.uint64(1)).astype(bool)


def numpy_rbm(n: int, edge_u, edge_v, edge_weight, seed: int, max_rounds: int = 10_000) -> OracleResult:
    """Restatement of rbm (matchers.py:357-410): per round every live vertex
    flips a coin; a blue vertex proposes along its max-key edge to a red
    neighbour, a red vertex accepts its max-key incoming proposal.  The key is
    local max's (weight, salt, edge id) with rerandomized salts; ranks from a
    lexsort of the live edges (tiebreak.py:92-102).  Raises RuntimeError after
    max_rounds rounds (RbmDidNotConverge)."""
    edge_u = np.asarray(edge_u, dtype=np.int64)
    edge_v = np.asarray(edge_v, dtype=np.int64)
    edge_weight = np.asarray(edge_weight, dtype=np.float64)
    prop = np.full(n, -1, dtype=np.int64)
    acc = np.full(n, -1, dtype=np.int64)
    done = np.zeros(n, dtype=bool)
    live = np.arange(edge_u.size, dtype=np.int64)
    parts, rounds = [], []
    r = 0
    while live.size:
        if r >= max_rounds:
            raise RuntimeError(f"no progress after {max_rounds} rounds")
        rs = round_seed(seed, r, True)
        order = np.lexsort((live, edge_salts(rs, live), edge_weight[live]))
        rank = np.empty(live.size, dtype=np.int64)
        rank[order] = np.arange(live.size, dtype=np.int64)
        us, vs = edge_u[live], edge_v[live]
        bu, bv = vertex_coins(rs, us), vertex_coins(rs, vs)
        fwd, bwd = bu & ~bv, bv & ~bu
        np.maximum.at(prop, us[fwd], rank[fwd])
        np.maximum.at(prop, vs[bwd], rank[bwd])
        pf = fwd & (prop[us] == rank)
        pb = bwd & (prop[vs] == rank)
        np.maximum.at(acc, vs[pf], rank[pf])
        np.maximum.at(acc, us[pb], rank[pb])
        won = (pf & (acc[vs] == rank)) | (pb & (acc[us] == rank))
        parts.append(live[won])
        done[us[won]] = True
        done[vs[won]] = True
        alive = ~(done[us] | done[vs])
        for ends in (us[alive], vs[alive]):
            prop[ends] = -1
            acc[ends] = -1
        rounds.append((int(live.size), int(won.sum()), int(live.size - alive.sum())))
        live = live[alive]
        r += 1
    matched = np.sort(np.concatenate(parts)) if parts else np.empty(0, dtype=np.int64)
    mate = np.full(n, -1, dtype=np.int64)
    if matched.size:
        mate[edge_u[matched]] = edge_v[matched]
        mate[edge_v[matched]] = edge_u[matched]
    return OracleResult(mate, matched, rounds)


# ---------------------------------------------------------------- generators

def build_graph_loop(edge_list, num_vertices=None):
    """graph.py:59-119 numbering contract, as (n, edge_u, edge_v, edge_weight)."""
    kept = {}
    us, vs, ws = [], [], []
    max_id = -1
    for pos, (u, v, w) in enumerate(edge_list):
        ui, vi = int(u), int(v)
        if ui < 0 or vi < 0:
            raise ValueError(f"edge {pos}: negative vertex id ({ui}, {vi})")
        if num_vertices is not None and (ui >= num_vertices or vi >= num_vertices):
            raise ValueError(f"edge {pos}: vertex id out of range")
        wf = float(w)
        if math.isnan(wf) or math.isinf(wf) or wf < 0.0:
            raise ValueError(f"edge {pos}: weight must be finite and >= 0, got {w!r}")
        if ui == vi:
            continue
        max_id = max(max_id, ui, vi)
        pair = (ui, vi) if ui < vi else (vi, ui)
        at = kept.get(pair)
        if at is None:
            kept[pair] = len(us)
            us.append(ui)
            vs.append(vi)
            ws.append(wf)
        elif wf > ws[at]:
            us[at], vs[at], ws[at] = ui, vi, wf
    n = num_vertices if num_vertices is not None else max_id + 1
    return (n, np.asarray(us, dtype=np.int64), np.asarray(vs, dtype=np.int64),
            np.asarray(ws, dtype=np.float64))


def gen_random_edges(n: int, alpha: int, seed: int):
    """generate.py:48-89 (sparse branch): raw (u, v, w) arrays before build."""
    if n < 2:
        raise ValueError("n must be >= 2")
    m = alpha * n
    capacity = n * (n - 1) // 2
    if m > capacity:
        raise ValueError("density infeasible")
    rng = np.random.default_rng(seed)
    if 2 * m > capacity:
        lo, hi = np.triu_indices(n, k=1)
        pick = rng.choice(capacity, size=m, replace=False)
        chosen = lo[pick] * n + hi[pick]
        weights = rng.random(m)
        return chosen // n, chosen % n, weights
    chosen = np.empty(0, dtype=np.int64)
    while chosen.size < m:
        need = m - chosen.size
        batch = need + need // 8 + 16
        a = rng.integers(0, n, size=batch, dtype=np.int64)
        b = rng.integers(0, n, size=batch, dtype=np.int64)
        ok = a != b
        lo = np.minimum(a[ok], b[ok])
        hi = np.maximum(a[ok], b[ok])
        packed = lo * n + hi
        _, first = np.unique(packed, return_index=True)
        packed = packed[np.sort(first)]
        packed = packed[~np.isin(packed, chosen)]
        chosen = np.concatenate([chosen, packed[:need]])
    weights = rng.random(m)
    return chosen // n, chosen % n, weights


def gen_random(n: int, alpha: int, seed: int, unit: bool = False):
    """generate.py:48-89 (+ with_unit_weights, :219-222).  The raw pairs are
    distinct and lo < hi, so build_graph keeps them in order unchanged."""
    u, v, w = gen_random_edges(n, alpha, seed)
    if unit:
        w = np.ones_like(w)
    return n, u.astype(np.int64), v.astype(np.int64), w.astype(np.float64)


def _morton_order(points: np.ndarray) -> np.ndarray:
    """generate.py:97-110."""
    q = np.clip((points * 65536.0).astype(np.uint32), 0, 65535).astype(np.uint64)

    def spread(b):
        b = (b | (b << np.uint64(16))) & np.uint64(0x0000FFFF0000FFFF)
        b = (b | (b << np.uint64(8))) & np.uint64(0x00FF00FF00FF00FF)
        b = (b | (b << np.uint64(4))) & np.uint64(0x0F0F0F0F0F0F0F0F)
        b = (b | (b << np.uint64(2))) & np.uint64(0x3333333333333333)
        b = (b | (b << np.uint64(1))) & np.uint64(0x5555555555555555)
        return b

    key = spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1))
    return np.argsort(key, kind="stable")


def _radius_edges_grid(points: np.ndarray, radius: float):
    """generate.py:146-197 (same cell sweep order, so same edge order)."""
    n = points.shape[0]
    side = max(1, int(math.floor(1.0 / radius)))
    cx = np.minimum((points[:, 0] / (1.0 / side)).astype(np.int64), side - 1)
    cy = np.minimum((points[:, 1] / (1.0 / side)).astype(np.int64), side - 1)
    cell = cx * side + cy
    order = np.lexsort((np.arange(n), cell))
    sorted_cell = cell[order]
    uniq, starts = np.unique(sorted_cell, return_index=True)
    starts = np.concatenate([starts, [n]])
    cell_slice = {int(c): (int(starts[i]), int(starts[i + 1])) for i, c in enumerate(uniq)}
    us, vs, ds = [], [], []
    r2 = radius * radius
    for i, c in enumerate(uniq):
        px, py = int(c) // side, int(c) % side
        own = order[starts[i]:starts[i + 1]]
        parts = []
        for dx in (-1, 0, 1):
            qx = px + dx
            if not 0 <= qx < side:
                continue
            for dy in (-1, 0, 1):
                qy = py + dy
                if not 0 <= qy < side:
                    continue
                sl = cell_slice.get(qx * side + qy)
                if sl is not None:
                    parts.append(order[sl[0]:sl[1]])
        cand = np.concatenate(parts)
        diff = points[own][:, None, :] - points[cand][None, :, :]
        d2 = np.einsum("ijk,ijk->ij", diff, diff)
        pi, qi = np.nonzero((d2 < r2) & (own[:, None] < cand[None, :]))
        if pi.size:
            us.append(own[pi])
            vs.append(cand[qi])
            ds.append(np.sqrt(d2[pi, qi]))
    if not us:
        e = np.empty(0, dtype=np.int64)
        return e, e.copy(), np.empty(0, dtype=np.float64)
    return np.concatenate(us), np.concatenate(vs), np.concatenate(ds)


def gen_rgg(x: int, seed: int, weight_mode: str = "euclidean"):
    """generate.py:113-143.  Raw pairs are distinct with u < v, so the
    build_graph numbering is the identity on the raw order."""
    n = 1 << x
    rng = np.random.default_rng(seed)
    points = rng.random((n, 2))
    points = points[_morton_order(points)]
    radius = 0.55 * math.sqrt(math.log(n) / n)
    eu, ev, dist = _radius_edges_grid(points, radius)
    w = dist if weight_mode == "euclidean" else rng.random(eu.size)
    return n, eu.astype(np.int64), ev.astype(np.int64), np.asarray(w, dtype=np.float64)


# ---------------------------------------------------------------- RMAT (new generator)

_RMAT_TAG0 = 0x524D41545F4C5654
_RMAT_TAG1 = 0x524D41545F574754
_RMAT_TAG2 = 0x524D41545F504552


def _mix64_int(x: int) -> int:
    return int(mix64(np.array([x & _UINT64_MASK], dtype=np.uint64))[0])


def rmat_perm(x: np.ndarray, scale: int, s2: int) -> np.ndarray:
    """Restatement of csrc/lmx_build.cu:rmat_perm (bijection on `scale` bits)."""
    mask = np.uint64((1 << scale) - 1)
    h = scale // 2 + 1
    h2 = scale - h if scale - h > 0 else 1
    with np.errstate(over="ignore"):
        y = x.astype(np.uint64)
        y = (y * np.uint64(0x9E3779B97F4A7C15)) & mask
        y ^= y >> np.uint64(h)
        y = (y * np.uint64(0xBF58476D1CE4E5B9)) & mask
        y ^= y >> np.uint64(h2)
        y ^= np.uint64(s2) & mask
    return y


def rmat_raw(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19, c: float = 0.19,
             seed: int = 1, permute: bool = True):
    """CPU restatement of the device RMAT generator (csrc/lmx_build.cu header)."""
    k = edge_factor << scale
    A = int(np.rint(a * 65536.0))
    B = int(np.rint(b * 65536.0))
    C = int(np.rint(c * 65536.0))
    AB, ABC = A + B, A + B + C
    s0 = _mix64_int((seed & _UINT64_MASK) ^ _RMAT_TAG0)
    s1 = _mix64_int((seed & _UINT64_MASK) ^ _RMAT_TAG1)
    s2 = _mix64_int((seed & _UINT64_MASK) ^ _RMAT_TAG2)
    i = np.arange(k, dtype=np.uint64)
    u = np.zeros(k, dtype=np.uint64)
    v = np.zeros(k, dtype=np.uint64)
    h = None
    with np.errstate(over="ignore"):
        for lvl in range(scale):
            if lvl % 4 == 0:
                h = mix64(np.uint64(s0) ^ (i * np.uint64(16) + np.uint64(lvl // 4)))
            x = (h >> np.uint64(16 * (lvl % 4))) & np.uint64(0xFFFF)
            bit = np.uint64(1 << (scale - 1 - lvl))
            ub = x >= np.uint64(AB)                                   # quadrants (1,0), (1,1)
            vb = ((x >= np.uint64(A)) & (x < np.uint64(AB))) | (x >= np.uint64(ABC))
            u |= np.where(ub, bit, np.uint64(0))
            v |= np.where(vb, bit, np.uint64(0))
        if permute:
            u = rmat_perm(u, scale, s2)
            v = rmat_perm(v, scale, s2)
        w = (mix64(np.uint64(s1) ^ i) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return u.astype(np.int64), v.astype(np.int64), w


def c_rmat_raw(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19, c: float = 0.19,
               seed: int = 1, permute: bool = True):
    """lmx_oracle.c:lmxo_rmat_raw -- rmat_raw with u32 ids, threaded, for scales
    numpy cannot hold (RMAT-26: 17 GB of raw triples)."""
    k = edge_factor << scale
    u = np.empty(k, dtype=np.uint32)
    v = np.empty(k, dtype=np.uint32)
    w = np.empty(k, dtype=np.float64)
    A = int(np.rint(a * 65536.0))
    B = int(np.rint(b * 65536.0))
    C = int(np.rint(c * 65536.0))
    _load().lmxo_rmat_raw(scale, k, A, A + B, A + B + C, seed & _UINT64_MASK, int(bool(permute)),
                          u.ctypes.data, v.ctypes.data, w.ctypes.data)
    return u, v, w


def c_build_graph(u, v, w, num_vertices: int):
    """lmx_oracle.c:lmxo_build_graph -- graph.py:59-119 on u32 raw triples
    (ids < num_vertices, weights valid) in O(k) extra memory.  Returns
    (n, edge_u int64, edge_v int64, edge_weight f64) views of capacity-k buffers."""
    u = np.ascontiguousarray(u, dtype=np.uint32)
    v = np.ascontiguousarray(v, dtype=np.uint32)
    w = np.ascontiguousarray(w, dtype=np.float64)
    k = int(u.size)
    rep = np.empty(max(k, 1), dtype=np.uint32)
    eu = np.empty(max(k, 1), dtype=np.int64)
    ev = np.empty(max(k, 1), dtype=np.int64)
    ew = np.empty(max(k, 1), dtype=np.float64)
    m = _load().lmxo_build_graph(k, u.ctypes.data, v.ctypes.data, w.ctypes.data, int(num_vertices),
                                 rep.ctypes.data, eu.ctypes.data, ev.ctypes.data, ew.ctypes.data)
    if m < 0:
        raise MemoryError("lmxo_build_graph: allocation failed")
    del rep
    return int(num_vertices), eu[:m], ev[:m], ew[:m]


def build_graph_vec(u, v, w, num_vertices=None):
    """Vectorised numpy restatement of graph.py:59-119 (pinned against
    build_graph_loop / the reference in tests); used for RMAT-size oracles."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    w = np.asarray(w, dtype=np.float64)
    pos = np.arange(u.size, dtype=np.int64)
    keep = u != v
    u, v, w, pos = u[keep], v[keep], w[keep], pos[keep]
    n = num_vertices if num_vertices is not None else (int(max(u.max(), v.max())) + 1 if u.size else 0)
    if u.size == 0:
        e = np.empty(0, dtype=np.int64)
        return n, e, e.copy(), np.empty(0, dtype=np.float64)
    lo = np.minimum(u, v)
    hi = np.maximum(u, v)
    key = lo * np.int64(max(n, 1)) + hi
    order = np.lexsort((pos, key))
    ks = key[order]
    head = np.ones(ks.size, dtype=bool)
    head[1:] = ks[1:] != ks[:-1]
    starts = np.nonzero(head)[0]
    run = np.cumsum(head) - 1
    ws = w[order]
    runmax = np.maximum.reduceat(ws, starts)
    is_max = ws == runmax[run]
    big = np.iinfo(np.int64).max
    cand = np.where(is_max, order, big)          # order is ascending inside a run
    kept = np.minimum.reduceat(cand, starts)
    first = order[starts]
    eo = np.argsort(first, kind="stable")
    kept = kept[eo]
    return n, u[kept], v[kept], w[kept]


# ---------------------------------------------------------------- coarsening (config C4, new)

_MESH_TAG = 0x4D4553485F444941


def mesh_edges(side: int, seed: int = 0):
    """Restatement of csrc/lmx_coarsen.cu:k_mesh (jittered-grid triangulation)."""
    s = side
    n = s * s
    v = np.arange(n, dtype=np.int64)
    i, j = v // s, v % s
    sm = _mix64_int((seed & _UINT64_MASK) ^ _MESH_TAG)
    main = (mix64(np.uint64(sm) ^ v.astype(np.uint64)) & np.uint64(1)).astype(bool)
    us, vs = [], []
    right = j + 1 < s
    down = i + 1 < s
    diag = right & down
    cnt = right.astype(np.int64) + down + diag
    off = np.concatenate([[0], np.cumsum(cnt)])
    m = int(off[-1])
    eu = np.empty(m, dtype=np.int64)
    ev = np.empty(m, dtype=np.int64)
    pos = off[:-1].copy()
    eu[pos[right]] = v[right]
    ev[pos[right]] = v[right] + 1
    pos += right
    eu[pos[down]] = v[down]
    ev[pos[down]] = v[down] + s
    pos += down
    a = np.where(main, v, v + 1)
    b = np.where(main, v + s + 1, v + s)
    eu[pos[diag]] = a[diag]
    ev[pos[diag]] = b[diag]
    return n, eu, ev, np.ones(m, dtype=np.float64)


def ratings(eu, ev, w, c):
    """Edge rating w(e)^2 / (c(u) c(v)) (the coarsening match weight)."""
    w = np.asarray(w, dtype=np.float64)
    return (w * w) / (c[eu] * c[ev])


def contract(n, eu, ev, w, c, mate):
    """Contraction rules of csrc/lmx_coarsen.cu: coarse ids by ascending
    representative (unmatched, or the smaller matched endpoint), summed node
    weights, parallel edges merged by summed weight in ascending (min, max)
    coarse-pair order."""
    v = np.arange(n, dtype=np.int64)
    rep_flag = (mate < 0) | (v < mate)
    scan = np.concatenate([[0], np.cumsum(rep_flag)])
    rep = np.where(rep_flag, v, mate)
    cid = scan[rep]
    nc = int(scan[-1])
    cc = np.bincount(cid, weights=c, minlength=nc)
    a, b = cid[eu], cid[ev]
    keep = a != b
    lo = np.minimum(a, b)[keep]
    hi = np.maximum(a, b)[keep]
    key = lo * np.int64(max(nc, 1)) + hi
    uk, inv = np.unique(key, return_inverse=True)
    cw = np.bincount(inv, weights=np.asarray(w, dtype=np.float64)[keep], minlength=uk.size)
    return nc, uk // max(nc, 1), uk % max(nc, 1), cw, cc, cid


def coarsen_levels(n, eu, ev, w, seed=0, min_n=1024, min_shrink=0.05, max_levels=64):
    """Reference pipeline for the C4 tests: per level (n, m, mate, matched ids, rounds)."""
    c = np.ones(n, dtype=np.float64)
    levels = []
    for lvl in range(max_levels):
        r = ratings(eu, ev, w, c)
        res = c_local_max(n, eu, ev, r, seed + lvl, True)
        levels.append((n, eu.size, res))
        nc, eu, ev, w, c, _ = contract(n, eu, ev, w, c, res.mate)
        if nc < min_n or (n - nc) < min_shrink * n:
            levels.append((nc, eu.size, None))
            break
        n = nc
    return levels


# ---------------------------------------------------------------- validate_matching (graph.py:212-237)

def validate_matching_loop(n: int, edge_u, edge_v, edge_ids, mate):
    """Loop restatement of ``validate_matching`` (graph.py:212-237): returns
    (valid, maximal).  The reference walks its frozenset; the flags do not
    depend on the order, so this walks the ids ascending."""
    mate = np.asarray(mate)
    if mate.shape != (n,):
        return False, False
    eu = np.asarray(edge_u)
    ev = np.asarray(edge_v)
    m = eu.size
    seen = np.zeros(n, dtype=bool)
    for k in sorted(int(x) for x in edge_ids):
        if not 0 <= k < m:
            return False, False
        u, v = int(eu[k]), int(ev[k])
        if seen[u] or seen[v]:
            return False, False
        seen[u] = seen[v] = True
        if mate[u] != v or mate[v] != u:
            return False, False
    if np.any(mate[~seen] != -1):
        return False, False
    addable = bool(np.any((mate[eu] == -1) & (mate[ev] == -1)))
    return True, not addable


# ---------------------------------------------------------------- partition_graph (bsp.py:60-98)

def partition_bounds(offsets, n: int, p: int) -> np.ndarray:
    """Restatement of partition_graph's cut points (bsp.py:67-83): contiguous
    ranges cut at the degree-prefix multiples of 2m/p, forced strictly
    increasing, each later worker left at least one vertex."""
    if p < 1:
        raise ValueError("p must be >= 1")
    if p > n:
        raise ValueError(f"p={p} exceeds the vertex count {n}")
    offsets = np.asarray(offsets, dtype=np.int64)
    two_m = int(offsets[-1])
    targets = (np.arange(1, p, dtype=np.float64) * two_m) / p
    cuts = np.searchsorted(offsets, targets, side="left").astype(np.int64)
    if cuts.size:
        steps = np.arange(1, p, dtype=np.int64)
        cuts = np.maximum.accumulate(cuts - steps) + steps
        cuts = np.minimum(np.maximum(cuts, steps), n - p + steps)
        return np.concatenate([[0], cuts, [n]]).astype(np.int64)
    return np.array([0, n], dtype=np.int64)


def bsp_messages(n: int, edge_u, edge_v, edge_weight, p: int, seed: int, rerandomize: bool = True):
    """Restatement of bsp_local_max's boundary accounting (bsp.py:148-199):
    per round, (round_index, candidate_records, bytes_estimate,
    cut_edges_surviving, status_records), over the live edge set of each round
    -- local_max_seq's (bsp.py:113-115), replayed by numpy_local_max's loop."""
    eu = np.asarray(edge_u, dtype=np.int64)
    ev = np.asarray(edge_v, dtype=np.int64)
    w = np.asarray(edge_weight, dtype=np.float64)
    deg = np.bincount(eu, minlength=n) + np.bincount(ev, minlength=n)
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(deg, out=offsets[1:])
    bounds = partition_bounds(offsets, n, p)
    owner = np.repeat(np.arange(p, dtype=np.int64), np.diff(bounds))
    is_cut = owner[eu] != owner[ev]
    cand_w = np.zeros(n, dtype=np.uint64)
    cand_s = np.zeros(n, dtype=np.uint64)
    cand_id = np.full(n, -1, dtype=np.int64)
    vm = np.zeros(n, dtype=bool)
    live = np.arange(eu.size, dtype=np.int64)
    out = []
    r = 0
    while live.size:
        cut_live = live[is_cut[live]]
        cu, cv = eu[cut_live], ev[cut_live]
        records = int(np.unique(cu * np.int64(p) + owner[cv]).size + np.unique(cv * np.int64(p) + owner[cu]).size)
        out.append((r, records, records * 32, int(cut_live.size), 2 * int(cut_live.size)))
        rs = round_seed(seed, r, rerandomize)
        wbits = weight_bits(w[live])
        salts = edge_salts(rs, live)
        us, vs = eu[live], ev[live]
        np.maximum.at(cand_w, us, wbits)
        np.maximum.at(cand_w, vs, wbits)
        tie_u = cand_w[us] == wbits
        tie_v = cand_w[vs] == wbits
        np.maximum.at(cand_s, us[tie_u], salts[tie_u])
        np.maximum.at(cand_s, vs[tie_v], salts[tie_v])
        tie_u &= cand_s[us] == salts
        tie_v &= cand_s[vs] == salts
        np.maximum.at(cand_id, us[tie_u], live[tie_u])
        np.maximum.at(cand_id, vs[tie_v], live[tie_v])
        won = (cand_id[us] == live) & (cand_id[vs] == live)
        vm[us[won]] = True
        vm[vs[won]] = True
        alive = ~(vm[us] | vm[vs])
        for ends in (us[alive], vs[alive]):
            cand_w[ends] = 0
            cand_s[ends] = 0
            cand_id[ends] = -1
        live = live[alive]
        r += 1
    return out
