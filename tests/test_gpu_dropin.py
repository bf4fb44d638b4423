"""Drop-in fidelity on the GPU:

* the one-shot C entry ``lmx_local_max`` through the exact ctypes binding
  INTEGRATION.md §2 tells a reference maintainer to add (the code block is
  executed from the markdown, so the document cannot drift), including a run
  with more rounds than its first ``rounds_out`` buffer;
* Python seeds outside [0, 2^64) (tiebreak.py:49 masks them);
* the device ``validate_matching`` against the unmodified reference's flags
  (tests/golden/validate.npz) and the oracle's loop restatement;
* results compare with ``==`` against the reference's own types when locmax
  is importable (baseline/_ref).
"""

from __future__ import annotations

import os
import re
import types

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _integration_binding():
    """Execute INTEGRATION.md §2's binding code block with the lib path set to ours."""
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = re.search(r"## 2\..*?```python\n(.*?)```", text, re.S).group(1)
    from paper_1302_4587_b200.engine import LIB_PATH
    block = block.replace('"/path/to/liblmx.so"', repr(LIB_PATH))
    # the binding's relative imports (`from .graph import ...`) resolve against
    # the reference package when it is importable, else against our mirrors
    try:
        import locmax.graph as lg
        import locmax.matchers as lm
        src = {"graph": lg, "matchers": lm}
    except ImportError:
        from paper_1302_4587_b200 import graph as pg
        src = {"graph": pg, "matchers": pg}
    block = block.replace("from .graph import", "from __lmx_graph__ import").replace(
        "from .matchers import", "from __lmx_matchers__ import")
    import sys
    sys.modules["__lmx_graph__"] = src["graph"]
    sys.modules["__lmx_matchers__"] = src["matchers"]
    mod = types.ModuleType("locmax_b200_binding")
    exec(compile(block, "INTEGRATION.md#2", "exec"), mod.__dict__)
    return mod


def _g(n, eu, ev, w):
    from paper_1302_4587_b200 import Graph
    return Graph(n, eu, ev, w)


@pytest.mark.parametrize("case", ["rmat", "unit", "rgg"])
def test_integration_binding_one_shot(case):
    mod = _integration_binding()
    if case == "rmat":
        u, v, w = O.rmat_raw(14, 16, seed=4, permute=True)
        n, eu, ev, ww = O.build_graph_vec(u, v, w, 1 << 14)
    elif case == "unit":
        n, eu, ev, ww = O.gen_random(1 << 14, 4, 9, unit=True)
    else:
        n, eu, ev, ww = O.gen_rgg(13, 2)
    g = _g(n, eu, ev, ww)
    m, trace = mod.local_max_b200(g, 5)
    ref = O.c_local_max(n, eu, ev, ww, 5, True)
    assert np.array_equal(np.asarray(m.mate), ref.mate)
    assert sorted(m.edges) == ref.matched_ids.tolist()
    assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in trace.rounds] == ref.rounds


def test_integration_binding_more_rounds_than_buffer():
    """A path with increasing weights needs ~n/2 rounds: more than the
    binding's first 64-entry rounds_out (LMX_ELIMIT -> retry with the size)."""
    mod = _integration_binding()
    n = 400
    eu = np.arange(n - 1, dtype=np.int64)
    ev = eu + 1
    w = np.arange(n - 1, dtype=np.float64) + 1.0
    g = _g(n, eu, ev, w)
    m, trace = mod.local_max_b200(g, 0)
    ref = O.c_local_max(n, eu, ev, w, 0, True)
    assert len(trace.rounds) == len(ref.rounds) > 64
    assert np.array_equal(np.asarray(m.mate), ref.mate)
    assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in trace.rounds] == ref.rounds


def test_integration_binding_value_error():
    mod = _integration_binding()
    g = _g(3, np.array([0, 1]), np.array([1, 2]), np.array([1.0, -2.0]))
    with pytest.raises(ValueError, match="weight"):
        mod.local_max_b200(g, 0)


@pytest.mark.parametrize("seed", [-1, -12345, 2 ** 64 + 7, 2 ** 63, 2 ** 64 - 1])
@pytest.mark.parametrize("rerandomize", [True, False])
def test_seeds_outside_u64_are_masked(seed, rerandomize):
    """tiebreak.py:49: round_seed masks the Python seed to 64 bits."""
    from paper_1302_4587_b200 import local_max_b200
    for n, eu, ev, w in (O.gen_random(3000, 4, 1, unit=True), O.gen_rgg(11, 1)):
        g = _g(n, eu, ev, w)
        m, trace = local_max_b200(g, seed, rerandomize)
        ref = O.c_local_max(n, eu, ev, w, seed, rerandomize)
        assert np.array_equal(np.asarray(m.mate), ref.mate)
        assert [(r.edges_before, r.edges_matched, r.edges_removed) for r in trace.rounds] == ref.rounds


def test_device_validate_equals_reference_flags(engine):
    """lmx_validate vs the unmodified reference's validate_matching flags
    (tests/golden/validate.npz) and the oracle's loop restatement."""
    from paper_1302_4587_b200 import Matching
    z = np.load(os.path.join(ROOT, "tests", "golden", "validate.npz"))
    for k in range(z["n"].size):
        n, alpha, seed = int(z["n"][k]), int(z["alpha"][k]), int(z["seed"][k])
        ids = z["ids"][z["ids_off"][k]:z["ids_off"][k + 1]]
        mate = z["mate"][z["mate_off"][k]:z["mate_off"][k + 1]]
        n_, eu, ev, w = O.gen_random(n, alpha, seed)
        engine.load_graph(_g(n_, eu, ev, w))
        got, _ = engine.validate(Matching(ids, mate))
        want = (bool(z["valid"][k]), bool(z["maximal"][k]))
        assert (got.valid, got.maximal) == want, (k, int(z["kind"][k]), got.detail)
        assert O.validate_matching_loop(n_, eu, ev, ids, mate) == want


def test_results_compare_with_reference_types():
    """With locmax importable, RoundStats IS locmax's and Matching subclasses it:
    ``==`` against the reference's own results holds in both directions."""
    lg = pytest.importorskip("locmax.graph")
    lm = pytest.importorskip("locmax.matchers")
    from paper_1302_4587_b200 import local_max_b200
    n, eu, ev, w = O.gen_random(2000, 4, 3)
    m, trace = local_max_b200(_g(n, eu, ev, w), 3)
    ref = O.c_local_max(n, eu, ev, w, 3, True)
    ref_m = lg.Matching(frozenset(ref.matched_ids.tolist()), ref.mate)
    ref_rounds = [lm.RoundStats(*r) for r in ref.rounds]
    assert isinstance(m, lg.Matching) and isinstance(trace, lm.PhaseTrace)
    assert m == ref_m and ref_m == m
    assert trace.rounds == ref_rounds
