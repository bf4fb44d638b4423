"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu`` and run on a B200
(``pytest -m gpu``); everything else runs on the CPU build box."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# The unmodified reference, when tools/install_reference.sh has put it in
# baseline/_ref: the drop-in then returns locmax's own result types, which is
# what the tests should see (never /root/reference: it is absent on the GPU box).
_REF = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(os.path.join(_REF, "locmax")) and _REF not in sys.path:
    sys.path.append(_REF)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running (large instances)")


@pytest.fixture(scope="session")
def golden_small():
    return np.load(os.path.join(GOLDEN, "small.npz"))


@pytest.fixture(scope="session")
def golden_instances():
    return np.load(os.path.join(GOLDEN, "instances.npz"))


@pytest.fixture(scope="session")
def golden_tiebreak():
    return np.load(os.path.join(GOLDEN, "tiebreak.npz"))


@pytest.fixture(scope="session")
def engine():
    from paper_1302_4587_b200 import Engine
    eng = Engine(0)
    yield eng
    eng.close()


def small_cases(z):
    """Yield (graph_index, n, raw (u, v, w), built (eu, ev, w), num_vertices_given)."""
    for gi in range(len(z["raw_off"]) - 1):
        a, b = z["raw_off"][gi], z["raw_off"][gi + 1]
        c, d = z["g_off"][gi], z["g_off"][gi + 1]
        gn = int(z["g_n"][gi])
        nv = None if gn >= 0 else -1 - gn
        n = gn if gn >= 0 else nv
        yield (gi, n, (z["raw_u"][a:b], z["raw_v"][a:b], z["raw_w"][a:b]),
               (z["g_u"][c:d], z["g_v"][c:d], z["g_w"][c:d]), nv)


def small_runs(z):
    """Yield (graph_index, seed, rerandomize, mate, ids, rounds) reference results."""
    for k in range(len(z["res_graph"])):
        ma, mb = z["res_mate_off"][k], z["res_mate_off"][k + 1]
        ia, ib = z["res_ids_off"][k], z["res_ids_off"][k + 1]
        ra, rb = z["res_rounds_off"][k], z["res_rounds_off"][k + 1]
        yield (int(z["res_graph"][k]), int(z["res_seed"][k]), bool(z["res_rr"][k]),
               z["res_mate"][ma:mb], z["res_ids"][ia:ib],
               [tuple(int(x) for x in row) for row in z["res_rounds"][ra:rb]])


INSTANCE_BUILDERS = {
    # name -> callable returning (n, eu, ev, w) via the oracle's restated generators
    "random-x16-a4-wunit-s0": lambda O: O.gen_random(1 << 16, 4, 0, unit=True),
    "random-x16-a4-wunit-s0-norr": lambda O: O.gen_random(1 << 16, 4, 0, unit=True),
    "random-x16-a4-s0": lambda O: O.gen_random(1 << 16, 4, 0),
    "rgg-x16-euclidean-s0": lambda O: O.gen_rgg(16, 0, "euclidean"),
    "rgg-x12-random-s3": lambda O: O.gen_rgg(12, 3, "random"),
    "random-x12-a16-s5": lambda O: O.gen_random(1 << 12, 16, 5),
    "random-x10-a200-dense-s1": lambda O: O.gen_random(1 << 10, 200, 1),
    "random-x20-a4-s1": lambda O: O.gen_random(1 << 20, 4, 1),
    "random-x20-a4-wunit-s2": lambda O: O.gen_random(1 << 20, 4, 2, unit=True),
}


def instance_graph(z, name):
    """(n, eu, ev, w) of a golden instance, regenerated (or stored for file-based ones)."""
    from oracle import oracle as O
    if f"{name}/edge_u" in z:
        return (int(z[f"{name}/n"]), z[f"{name}/edge_u"].astype(np.int64),
                z[f"{name}/edge_v"].astype(np.int64), z[f"{name}/edge_weight"])
    return INSTANCE_BUILDERS[name](O)


def edges_digest(eu, ev, w) -> str:
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(eu, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(ev, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(w, dtype="<f8").view("<u8").tobytes())
    return h.hexdigest()[:32]


def mate_digest(mate) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(mate, dtype="<i8").tobytes()).hexdigest()[:16]
