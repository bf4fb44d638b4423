"""Generate the golden fixtures in this directory from the UNMODIFIED reference.

Run in the build container (the reference exists only there):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (all small, committed):
  tiebreak.npz   -- mix64 / round_seed / edge_salts / weight_bits vectors
                    (tiebreak.py:28-59,105-113)
  small.npz      -- ~400 small graphs (raw edge lists incl. self-loops,
                    duplicates, -0.0, ties) with reference build_graph output
                    (graph.py:59-119) and local_max_seq results
                    (matchers.py:61-122) for several seeds, both rerandomize
                    settings
  instances.npz  -- reference-generated instances (gen_random, gen_rgg,
                    with_unit_weights, the delaunay_x10 fixture): sha256 of
                    the edge arrays, full mate arrays for x<=16, digests,
                    round traces and matching weights
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

from locmax import build_graph, gen_random, gen_rgg, local_max_seq, read_graph
from locmax.generate import with_unit_weights
from locmax.tiebreak import edge_salts, mix64, round_seed, weight_bits

HERE = os.path.dirname(os.path.abspath(__file__))


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).hexdigest()[:16]


def edges_digest(g) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(g.edge_u, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(g.edge_v, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(g.edge_weight, dtype="<f8").view("<u8").tobytes())
    return h.hexdigest()[:32]


def make_tiebreak() -> None:
    vals = np.array([0, 1, 2, 3, 255, 2**32 - 1, 2**32, 2**63, 2**64 - 1,
                     0x123456789ABCDEF0, 0xDEADBEEFCAFEBABE], dtype=np.uint64)
    rng = np.random.default_rng(123)
    vals = np.concatenate([vals, rng.integers(0, 2**63, size=200, dtype=np.uint64) * np.uint64(2)
                           + rng.integers(0, 2, size=200, dtype=np.uint64)])
    seeds = [0, 1, 2, 3, 5, 7, 42, 12345, 2**31 - 1, 2**32, 2**63, 2**64 - 1, 2**64 + 7, -1, -12345]
    rs_rows = []
    for s in seeds:
        for r in range(0, 14):
            for flag in (True, False):
                rs_rows.append((s & (2**64 - 1), r, int(flag), round_seed(s, r, flag)))
    rs_arr = np.array([[a, b, c, d] for a, b, c, d in rs_rows], dtype=np.uint64)
    ids = np.concatenate([np.arange(0, 1000, dtype=np.uint64),
                          np.array([2**32 - 1, 2**32, 2**33 + 5, 2**40], dtype=np.uint64)])
    salt_seeds = np.array([round_seed(0, 0), round_seed(0, 1), round_seed(7, 3),
                           round_seed(-1, 0)], dtype=np.uint64)
    salts = np.stack([edge_salts(int(s), ids) for s in salt_seeds])
    w = np.array([-0.0, 0.0, 1.0, 0.5, 1e-300, 5e-324, 0.999999999, 1e300, 2.0, 3.0], dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, "tiebreak.npz"),
                        mix_in=vals, mix_out=mix64(vals.copy()),
                        rs=rs_arr, salt_ids=ids, salt_seeds=salt_seeds, salts=salts,
                        wb_in=w, wb_out=weight_bits(w))


def random_edge_list(rng, n, m, mode):
    """Raw edge lists exercising build_graph: self-loops, duplicates with
    heavier/lighter/equal weights in either orientation, -0.0, ties."""
    out = []
    for _ in range(m):
        u = int(rng.integers(0, n))
        v = int(rng.integers(0, n)) if rng.random() > 0.05 else u
        if mode == 0:
            w = float(rng.random())
        elif mode == 1:
            w = float(rng.integers(1, 4))
        elif mode == 2:
            w = 1.0
        else:
            w = float(rng.choice([0.0, -0.0, 0.5, 1.0]))
        out.append((u, v, w))
    return out


def make_small() -> None:
    rng = np.random.default_rng(2024)
    raw_u, raw_v, raw_w, raw_off = [], [], [], [0]
    g_n, g_off, g_u, g_v, g_w = [], [0], [], [], []
    res_graph, res_seed, res_rr = [], [], []
    res_mate, res_mate_off = [], [0]
    res_ids, res_ids_off = [], [0]
    res_rounds, res_rounds_off = [], [0]
    cases = []
    cases.append(([(0, 1, 1.0), (1, 2, 2.0), (0, 2, 3.0)], None))           # triangle
    cases.append(([(0, 1, 2.0), (1, 2, 3.0), (2, 3, 2.0)], None))           # path4
    cases.append(([(0, leaf, 1.0) for leaf in range(1, 9)], None))          # star9
    cases.append(([(0, 1, 0.0), (1, 2, 0.0), (2, 3, 0.0), (3, 0, 0.0)], None))  # zero 4-cycle
    cases.append(([], 4))                                                   # edgeless
    cases.append(([(0, 1, 1.0)], None))
    cases.append(([(0, 1, -0.0), (1, 2, 0.0), (2, 0, -0.0)], None))
    cases.append(([(3, 1, 1.0), (1, 3, 2.0), (1, 3, 2.0), (2, 2, 5.0), (0, 2, 1.0)], None))
    cases.append(([(u, v, 1.0) for u, v in zip(*np.triu_indices(12, k=1))], None))  # K12 unit
    for i in range(400):
        n = int(rng.integers(2, 40))
        m = int(rng.integers(0, 3 * n + 1))
        cases.append((random_edge_list(rng, n, m, i % 4), n if i % 3 else None))
    for gi, (edges, nv) in enumerate(cases):
        g = build_graph(edges, num_vertices=nv)
        for (u, v, w) in edges:
            raw_u.append(u); raw_v.append(v); raw_w.append(w)
        raw_off.append(len(raw_u))
        g_n.append(g.num_vertices if nv is None else -1 - nv)  # negative: n was given
        g_u.extend(g.edge_u.tolist()); g_v.extend(g.edge_v.tolist()); g_w.extend(g.edge_weight.tolist())
        g_off.append(len(g_u))
        seeds = [0, gi, 7 * gi + 3] if gi % 2 == 0 else [gi]
        for seed in seeds:
            for flag in (True, False):
                mt, tr = local_max_seq(g, seed, flag)
                res_graph.append(gi); res_seed.append(seed); res_rr.append(int(flag))
                res_mate.extend(mt.mate.tolist()); res_mate_off.append(len(res_mate))
                res_ids.extend(mt.sorted_edge_ids().tolist()); res_ids_off.append(len(res_ids))
                for r in tr.rounds:
                    res_rounds.append((r.edges_before, r.edges_matched, r.edges_removed))
                res_rounds_off.append(len(res_rounds))
    np.savez_compressed(
        os.path.join(HERE, "small.npz"),
        raw_u=np.array(raw_u, dtype=np.int64), raw_v=np.array(raw_v, dtype=np.int64),
        raw_w=np.array(raw_w, dtype=np.float64), raw_off=np.array(raw_off, dtype=np.int64),
        g_n=np.array(g_n, dtype=np.int64), g_off=np.array(g_off, dtype=np.int64),
        g_u=np.array(g_u, dtype=np.int64), g_v=np.array(g_v, dtype=np.int64),
        g_w=np.array(g_w, dtype=np.float64),
        res_graph=np.array(res_graph, dtype=np.int64), res_seed=np.array(res_seed, dtype=np.int64),
        res_rr=np.array(res_rr, dtype=np.int64),
        res_mate=np.array(res_mate, dtype=np.int64), res_mate_off=np.array(res_mate_off, dtype=np.int64),
        res_ids=np.array(res_ids, dtype=np.int64), res_ids_off=np.array(res_ids_off, dtype=np.int64),
        res_rounds=np.array(res_rounds, dtype=np.int64).reshape(-1, 3),
        res_rounds_off=np.array(res_rounds_off, dtype=np.int64),
    )
    print("small cases:", len(cases), "runs:", len(res_graph))


def make_instances() -> None:
    specs = [
        # name, builder, seed, rerandomize, keep full mate
        ("random-x16-a4-wunit-s0", lambda: with_unit_weights(gen_random(1 << 16, 4, 0)), 0, True, True),
        ("random-x16-a4-wunit-s0-norr", lambda: with_unit_weights(gen_random(1 << 16, 4, 0)), 0, False, True),
        ("random-x16-a4-s0", lambda: gen_random(1 << 16, 4, 0), 0, True, True),
        ("rgg-x16-euclidean-s0", lambda: gen_rgg(16, 0, "euclidean"), 0, True, True),
        ("rgg-x12-random-s3", lambda: gen_rgg(12, 3, "random"), 3, True, True),
        ("random-x12-a16-s5", lambda: gen_random(1 << 12, 16, 5), 5, True, True),
        ("random-x10-a200-dense-s1", lambda: gen_random(1 << 10, 200, 1), 1, True, True),
        ("delaunay_x10", lambda: read_graph("/root/reference/pkg/tests/fixtures/delaunay_x10.txt"), 0, True, True),
        ("delaunay_x10-unit", lambda: with_unit_weights(
            read_graph("/root/reference/pkg/tests/fixtures/delaunay_x10.txt")), 4, True, True),
        ("random-x20-a4-s1", lambda: gen_random(1 << 20, 4, 1), 1, True, False),
        ("random-x20-a4-wunit-s2", lambda: with_unit_weights(gen_random(1 << 20, 4, 2)), 2, True, False),
    ]
    out = {}
    names = []
    for name, builder, seed, flag, full in specs:
        g = builder()
        mt, tr = local_max_seq(g, seed, flag)
        names.append(name)
        out[f"{name}/n"] = np.int64(g.num_vertices)
        out[f"{name}/m"] = np.int64(g.num_edges)
        out[f"{name}/edges_sha"] = np.array(edges_digest(g))
        out[f"{name}/seed"] = np.int64(seed)
        out[f"{name}/rerandomize"] = np.int64(int(flag))
        out[f"{name}/mate_digest"] = np.array(digest(mt.mate))
        out[f"{name}/size"] = np.int64(mt.size)
        out[f"{name}/weight"] = np.float64(mt.weight(g))
        out[f"{name}/rounds"] = np.array(
            [(r.edges_before, r.edges_matched, r.edges_removed) for r in tr.rounds], dtype=np.int64)
        if full:
            out[f"{name}/mate"] = mt.mate.astype(np.int32)
        if name.startswith("delaunay"):
            out[f"{name}/edge_u"] = g.edge_u.astype(np.int32)
            out[f"{name}/edge_v"] = g.edge_v.astype(np.int32)
            out[f"{name}/edge_weight"] = g.edge_weight
        print(name, g.num_vertices, g.num_edges, mt.size, len(tr.rounds), digest(mt.mate))
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "instances.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["tiebreak", "small", "instances"]
    if "tiebreak" in which:
        make_tiebreak()
    if "small" in which:
        make_small()
    if "instances" in which:
        make_instances()
