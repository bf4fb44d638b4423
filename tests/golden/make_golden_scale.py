"""Scale fixtures: digests of the reference matching on the BASELINE configs.

TEST INFRASTRUCTURE.  Run in the build container (CPU only):

    python tests/golden/make_golden_scale.py [--configs rmat24,rmat26,rgg22] \
        [--reference /root/reference/pkg/src]

For every config the input graph is generated on the CPU by the oracle's
restatements (never by the CUDA engine), matched by the pinned C oracle
(oracle/lmx_oracle.c, a restatement of matchers.py:61-122), and summarised in
``scale.json``:

* ``edges``   -- sha256 prefix of (edge_u, edge_v, edge_weight bits), the
                 format of make_golden.py's ``edges_digest``;
* ``mate``    -- sha256 of the little-endian int64 mate array (full hex);
* ``ids``     -- sha256 of the ascending matched edge ids (int64);
* ``rounds``  -- the RoundStats trace (edges_before, edges_matched, edges_removed);
* ``weight``  -- Matching.weight (graph.py:54-56: edge_weight[sorted ids].sum()),
                 as the float's hex so it compares bit for bit.

With ``--reference`` the UNMODIFIED reference is imported and, where it fits
this container's memory, run on the same arrays: ``locmax.local_max_seq``
(matchers.py:61-122) must give the identical mate / ids / trace / weight
(``reference_checked``), and for rgg22 ``locmax.gen_rgg`` must give the
identical graph (``generator_checked``).  RMAT-26 (~170 GB for the
reference) is matched by the C oracle alone.

Configs (BASELINE.json configs / north_star):
  rgg22   C2: gen_rgg(22, seed=0, "euclidean") (generate.py:113-143), match seed 0
  rmat24  C3: RMAT scale 24 ef 16 (.57,.19,.19), graph seed 1, permuted; match seed 1
  rmat26  N*: RMAT scale 26, same recipe (the bench workload)
  rmat27  RMAT scale 27, same recipe (2.1 G edges, the largest graph one B200
          holds; ~70 GB of host memory: made on a GPU box's host, whose 196 GB
          fit it, with `gpurun -- python tests/golden/make_golden_scale.py
          --configs rmat27`; C oracle only)
  er24unit C1 family at 256x: 4 * 2^24 uniform raw pairs (the RMAT generator
          with a = b = c = 1/4, no relabelling), unit weights; seed 1
  er24unit-norr  the same graph and seed, rerandomize=False
"""

from __future__ import annotations

import argparse
import gc
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

OUT = os.path.join(HERE, "scale.json")
RMAT_ABC = (0.57, 0.19, 0.19)


def sha(a: np.ndarray, dtype="<i8") -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=dtype).data).hexdigest()


def edges_digest(eu, ev, w) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(eu, dtype="<i8").data)
    h.update(np.ascontiguousarray(ev, dtype="<i8").data)
    h.update(np.ascontiguousarray(w, dtype="<f8").view("<u8").data)
    return h.hexdigest()[:32]


def summarise(name, n, eu, ev, w, seed, rerandomize=True, **extra):
    t0 = time.time()
    res = O.c_local_max(n, eu, ev, w, seed, rerandomize)
    t_match = time.time() - t0
    weight = float(np.asarray(w)[res.matched_ids].sum()) if res.matched_ids.size else 0.0
    rec = {
        "n": int(n), "m": int(eu.size), "seed": seed, "rerandomize": rerandomize,
        "edges": edges_digest(eu, ev, w),
        "mate": sha(res.mate), "ids": sha(res.matched_ids), "matched": int(res.matched_ids.size),
        "rounds": [list(r) for r in res.rounds], "weight": weight.hex(),
        "oracle_match_s": round(t_match, 1),
    }
    rec.update(extra)
    print(f"{name}: n={n} m={eu.size} |M|={res.matched_ids.size} rounds={len(res.rounds)} "
          f"match {t_match:.1f}s", flush=True)
    return rec, res


def check_reference(name, n, eu, ev, w, seed, rec, res, rerandomize=True):
    """Run the unmodified locmax.local_max_seq on the same arrays."""
    from locmax.graph import Graph
    from locmax.matchers import local_max_seq
    empty = np.empty(0, dtype=np.int64)
    g = Graph(int(n), np.zeros(n + 1, dtype=np.int64), empty, empty,
              np.asarray(eu, dtype=np.int64), np.asarray(ev, dtype=np.int64), np.asarray(w, dtype=np.float64))
    t0 = time.time()
    mm, tr = local_max_seq(g, seed, rerandomize)
    dt = time.time() - t0
    ids = np.array(sorted(mm.edges), dtype=np.int64)
    same = (np.array_equal(np.asarray(mm.mate), res.mate) and np.array_equal(ids, res.matched_ids)
            and [(r.edges_before, r.edges_matched, r.edges_removed) for r in tr.rounds] == res.rounds
            and float(mm.weight(g)).hex() == rec["weight"])
    print(f"{name}: reference local_max_seq {dt:.1f}s, identical: {same}", flush=True)
    if not same:
        raise SystemExit(f"{name}: the C oracle disagrees with the reference")
    rec["reference_checked"] = True
    rec["reference_s"] = round(dt, 1)


def make_rmat(scale, ref):
    t0 = time.time()
    u, v, w = O.c_rmat_raw(scale, 16, *RMAT_ABC, seed=1, permute=True)
    n, eu, ev, ew = O.c_build_graph(u, v, w, 1 << scale)
    del u, v, w
    gc.collect()
    print(f"rmat{scale}: generated + built in {time.time() - t0:.1f}s", flush=True)
    rec, res = summarise(f"rmat{scale}", n, eu, ev, ew, 1, graph_seed=1, permuted=True,
                         recipe=f"RMAT scale {scale} ef 16 (a,b,c)={RMAT_ABC}")
    if ref and scale <= 24:
        check_reference(f"rmat{scale}", n, eu, ev, ew, 1, rec, res)
    return rec


def make_er24unit(ref, rerandomize=True):
    t0 = time.time()
    u, v, w = O.c_rmat_raw(24, 4, 0.25, 0.25, 0.25, seed=1, permute=False)
    w[:] = 1.0
    n, eu, ev, ew = O.c_build_graph(u, v, w, 1 << 24)
    del u, v, w
    gc.collect()
    name = "er24unit" if rerandomize else "er24unit-norr"
    print(f"{name}: generated + built in {time.time() - t0:.1f}s", flush=True)
    rec, res = summarise(name, n, eu, ev, ew, 1, rerandomize, graph_seed=1, permuted=False,
                         recipe="4 * 2^24 uniform pairs (RMAT a=b=c=1/4), unit weights")
    if ref:
        check_reference(name, n, eu, ev, ew, 1, rec, res, rerandomize)
    return rec


def make_rgg22(ref):
    t0 = time.time()
    n, eu, ev, w = O.gen_rgg(22, 0, "euclidean")
    print(f"rgg22: oracle generator {time.time() - t0:.1f}s", flush=True)
    rec, res = summarise("rgg22", n, eu, ev, w, 0, graph_seed=0, recipe="gen_rgg(22, 0, 'euclidean')")
    if ref:
        from locmax.generate import gen_rgg
        t0 = time.time()
        g = gen_rgg(22, 0, "euclidean")
        same = edges_digest(g.edge_u, g.edge_v, g.edge_weight) == rec["edges"] and g.num_vertices == n
        print(f"rgg22: reference generator {time.time() - t0:.1f}s, identical: {same}", flush=True)
        if not same:
            raise SystemExit("rgg22: the oracle generator disagrees with the reference")
        rec["generator_checked"] = True
        del g
        gc.collect()
        check_reference("rgg22", n, eu, ev, w, 0, rec, res)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="rgg22,rmat24,rmat26")
    ap.add_argument("--reference", default=None, help="path of the reference's src/ (imports locmax)")
    args = ap.parse_args()
    if args.reference:
        sys.path.insert(0, args.reference)
    O.build()
    out = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            out = json.load(f)
    for name in args.configs.split(","):
        if name == "rgg22":
            out[name] = make_rgg22(bool(args.reference))
        elif name == "er24unit":
            out[name] = make_er24unit(bool(args.reference))
        elif name == "er24unit-norr":
            out[name] = make_er24unit(bool(args.reference), rerandomize=False)
        elif name.startswith("rmat"):
            out[name] = make_rmat(int(name[4:]), bool(args.reference))
        else:
            raise SystemExit(f"unknown config {name}")
        with open(OUT, "w") as f:
            json.dump(out, f, indent=1, sort_keys=True)
        gc.collect()


if __name__ == "__main__":
    main()
