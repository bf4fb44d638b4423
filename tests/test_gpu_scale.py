"""Bit-exact parity at the BASELINE configs' full sizes.

tests/golden/scale.json holds, per config, the digests of the graph and of
the reference matching, made on the CPU by tests/golden/make_golden_scale.py
(oracle generators + the pinned C oracle of matchers.py:61-122; for rgg22 and
rmat24 also checked identical to the unmodified locmax generator and
local_max_seq).  Here the graph is produced as the product produces it (the
device RMAT generator + build_graph; for C2 the host restatement of
generate.py's RGG loaded through the public API), matched on the B200, and
every digest compared: edge arrays, mate, matched ids, RoundStats, weight.
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(ROOT, "tests", "golden", "scale.json")) as _f:
    SCALE = json.load(_f)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").data).hexdigest()


def _edges(eu, ev, w):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(eu, dtype="<i8").data)
    h.update(np.ascontiguousarray(ev, dtype="<i8").data)
    h.update(np.ascontiguousarray(w, dtype="<f8").view("<u8").data)
    return h.hexdigest()[:32]


def _check(want, g, mate, ids, rounds):
    assert g.num_vertices == want["n"] and g.num_edges == want["m"]
    assert _edges(g.edge_u, g.edge_v, g.edge_weight) == want["edges"], "graph differs"
    assert [[r.edges_before, r.edges_matched, r.edges_removed] for r in rounds] == want["rounds"]
    assert ids.size == want["matched"]
    assert _sha(mate) == want["mate"], "mate differs"
    assert _sha(ids) == want["ids"], "matched ids differ"
    weight = float(np.asarray(g.edge_weight)[ids].sum()) if ids.size else 0.0
    assert weight.hex() == want["weight"], "Matching.weight differs"


@pytest.mark.parametrize("name", ["rmat24", "rmat26"])
def test_rmat_full_size_bit_exact(engine, name):
    want = SCALE[name]
    scale = int(name[4:])
    engine.gen_rmat(scale, 16, 0.57, 0.19, 0.19, seed=want["graph_seed"], permute=True)
    mate, ids, rounds = engine.match_raw(want["seed"], want["rerandomize"])
    g = engine.export_graph()
    _check(want, g, mate, ids, rounds)


def test_rgg22_c2_bit_exact(engine):
    """BASELINE config C2: gen_rgg(22, seed=0, "euclidean"), match seed 0."""
    from oracle import oracle as O
    from paper_1302_4587_b200 import Graph
    want = SCALE["rgg22"]
    n, eu, ev, w = O.gen_rgg(22, want["graph_seed"], "euclidean")
    g = Graph(n, eu, ev, w)
    engine.load_graph(g)
    mate, ids, rounds = engine.match_raw(want["seed"], want["rerandomize"])
    _check(want, g, mate, ids, rounds)


def test_er24_unit_weights_bit_exact(engine):
    """The C1 family at 256x (bench workload er24unit): unit weights, so the
    salts decide every round -- the compacting loop; pinned to the unmodified
    local_max_seq when the fixture was made."""
    want = SCALE["er24unit"]
    engine.gen_er(24, 4, seed=want["graph_seed"], unit=True)
    assert engine.algo() == "compact" and engine.layout() == "uniform"
    mate, ids, rounds = engine.match_raw(want["seed"], want["rerandomize"])
    _check(want, engine.export_graph(), mate, ids, rounds)


def test_er24_unit_static_order_bit_exact(engine):
    """The same graph with rerandomize=False (er24unit-norr, pinned to the
    unmodified local_max_seq): the static (weight, salt) layout on the scan
    loop, and the compacting loop, both equal the reference."""
    want = SCALE["er24unit-norr"]
    assert want["rerandomize"] is False and want.get("reference_checked")
    engine.set_static_order(want["seed"])
    engine.gen_er(24, 4, seed=want["graph_seed"], unit=True)
    engine.set_static_order(None)
    assert engine.algo() == "scan" and engine.static_order()
    mate, ids, rounds = engine.match_raw(want["seed"], False)
    g = engine.export_graph()
    _check(want, g, mate, ids, rounds)
    engine.load_graph(g)                                   # no static order: the compacting loop
    assert engine.algo() == "compact"
    mate, ids, rounds = engine.match_raw(want["seed"], False)
    _check(want, g, mate, ids, rounds)


@pytest.mark.parametrize("name,x,seed,mode", [("rgg-x16-euclidean-s0", 16, 0, "euclidean"),
                                               ("rgg-x12-random-s3", 12, 3, "random")])
def test_device_rgg_generator_equals_reference(engine, golden_instances, name, x, seed, mode):
    """lmx_gen_rgg reproduces the unmodified reference's gen_rgg graph (the
    reference's edge-array digest in tests/golden/instances.npz) and its
    matching."""
    from conftest import edges_digest, mate_digest
    z = golden_instances
    engine.gen_rgg(x, seed, mode)
    g = engine.export_graph()
    assert g.num_vertices == int(z[f"{name}/n"]) and g.num_edges == int(z[f"{name}/m"])
    assert edges_digest(g.edge_u, g.edge_v, g.edge_weight) == str(z[f"{name}/edges_sha"])
    mate, ids, rounds = engine.match_raw(int(z[f"{name}/seed"]), bool(z[f"{name}/rerandomize"]))
    assert mate_digest(mate) == str(z[f"{name}/mate_digest"])


def test_device_rgg22_c2(engine):
    """BASELINE config C2 built on the device: the graph the reference's
    gen_rgg(22, 0) builds (scale.json, generator_checked), and its matching."""
    want = SCALE["rgg22"]
    engine.gen_rgg(22, want["graph_seed"], "euclidean")
    mate, ids, rounds = engine.match_raw(want["seed"], want["rerandomize"])
    _check(want, engine.export_graph(), mate, ids, rounds)
