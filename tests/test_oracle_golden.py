"""Pin the CPU oracle (oracle/) to the reference's own outputs (tests/golden,
generated from the unmodified reference by tests/golden/make_golden.py)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import edges_digest, instance_graph, mate_digest, small_cases, small_runs
from oracle import oracle as O


def test_mix64_matches_reference(golden_tiebreak):
    z = golden_tiebreak
    assert np.array_equal(O.mix64(z["mix_in"]), z["mix_out"])
    for x, y in list(zip(z["mix_in"], z["mix_out"]))[:40]:
        assert O.c_mix64(int(x)) == int(y)


def test_round_seed_matches_reference(golden_tiebreak):
    for s, r, flag, want in golden_tiebreak["rs"]:
        assert O.round_seed(int(s), int(r), bool(flag)) == int(want)
        assert O.c_round_seed(int(s), int(r), bool(flag)) == int(want)


def test_survey_appendix_b_values():
    # SURVEY.md Appendix B, generated from the reference
    assert [O.c_mix64(x) for x in (0, 1, 2**64 - 1)] == [
        0xE220A8397B1DCDAF, 0x910A2DEC89025CC1, 0xE4D971771B652C20]
    assert O.round_seed(0, 0) == 0xA706DD2F4D197E6F
    assert O.round_seed(0, 1) == 0x08B4FDA8C892B50E
    assert O.round_seed(0, 5, rerandomize=False) == 0xA706DD2F4D197E6F
    assert O.round_seed(7, 3) == 0x6BAA78681A99F995
    assert O.round_seed(-1, 0) == 0x5DC20AA7B2A27137
    assert O.round_seed(2**64 + 7, 0) == 0xB8B4C2977EABCE45


def test_edge_salts_match_reference(golden_tiebreak):
    z = golden_tiebreak
    for rs, row in zip(z["salt_seeds"], z["salts"]):
        assert np.array_equal(O.edge_salts(int(rs), z["salt_ids"]), row)
        assert np.array_equal(O.c_edge_salts(int(rs), z["salt_ids"]), row)


def test_weight_bits_match_reference(golden_tiebreak):
    z = golden_tiebreak
    assert np.array_equal(O.weight_bits(z["wb_in"]), z["wb_out"])


def test_build_graph_restatements_match_reference(golden_small):
    for gi, n, raw, built, nv in small_cases(golden_small):
        for got in (O.build_graph_loop(list(zip(*raw)), nv), O.build_graph_vec(*raw, nv)):
            gn, eu, ev, w = got
            assert gn == n, gi
            assert np.array_equal(eu, built[0]) and np.array_equal(ev, built[1]), gi
            assert np.array_equal(w.view(np.uint64), built[2].view(np.uint64)), gi


@pytest.mark.parametrize("impl", ["c", "numpy"])
def test_oracle_local_max_matches_reference_small(golden_small, impl):
    graphs = {gi: (n, built) for gi, n, _, built, _ in small_cases(golden_small)}
    fn = O.c_local_max if impl == "c" else O.numpy_local_max
    count = 0
    for gi, seed, rr, mate, ids, rounds in small_runs(golden_small):
        n, (eu, ev, w) = graphs[gi]
        res = fn(n, eu, ev, w, seed, rr)
        assert np.array_equal(res.mate, mate), (gi, seed, rr)
        assert np.array_equal(res.matched_ids, ids), (gi, seed, rr)
        assert res.rounds == rounds, (gi, seed, rr)
        count += 1
    assert count > 1000


FAST_INSTANCES = ["random-x16-a4-wunit-s0", "random-x16-a4-wunit-s0-norr", "random-x16-a4-s0",
                  "rgg-x12-random-s3", "random-x12-a16-s5", "random-x10-a200-dense-s1",
                  "delaunay_x10", "delaunay_x10-unit"]


@pytest.mark.parametrize("name", FAST_INSTANCES)
def test_oracle_matches_reference_instances(golden_instances, name):
    z = golden_instances
    n, eu, ev, w = instance_graph(z, name)
    assert n == int(z[f"{name}/n"]) and eu.size == int(z[f"{name}/m"])
    assert edges_digest(eu, ev, w) == str(z[f"{name}/edges_sha"])
    res = O.c_local_max(n, eu, ev, w, int(z[f"{name}/seed"]), bool(z[f"{name}/rerandomize"]))
    assert mate_digest(res.mate) == str(z[f"{name}/mate_digest"])
    if f"{name}/mate" in z:
        assert np.array_equal(res.mate, z[f"{name}/mate"].astype(np.int64))
    assert [list(r) for r in res.rounds] == z[f"{name}/rounds"].tolist()
    assert res.matched_ids.size == int(z[f"{name}/size"])
    assert float(w[res.matched_ids].sum()) == float(z[f"{name}/weight"])


def test_survey_c1_golden():
    # |M| = 29 214, 5 rounds, mate digest 34039b07576f826f
    n, eu, ev, w = O.gen_random(1 << 16, 4, 0, unit=True)
    res = O.c_local_max(n, eu, ev, w, 0, True)
    assert res.matched_ids.size == 29214
    assert len(res.rounds) == 5
    assert res.rounds[0] == (262144, 16459, 202994)
    assert mate_digest(res.mate) == "34039b07576f826f"


def test_rmat_raw_is_deterministic_and_in_range():
    u, v, w = O.rmat_raw(8, 4, seed=3)
    u2, v2, w2 = O.rmat_raw(8, 4, seed=3)
    assert np.array_equal(u, u2) and np.array_equal(v, v2) and np.array_equal(w, w2)
    assert u.min() >= 0 and u.max() < 256 and v.min() >= 0 and v.max() < 256
    assert (w >= 0).all() and (w < 1).all()
    # permutation is a bijection on the id space
    assert np.unique(O.rmat_perm(np.arange(256), 8, 12345)).size == 256


def test_validate_loop_matches_reference_flags():
    """oracle.validate_matching_loop vs the unmodified reference's
    validate_matching (tests/golden/validate.npz, make_golden_validate.py)."""
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "validate.npz"))
    for k in range(z["n"].size):
        n, eu, ev, w = O.gen_random(int(z["n"][k]), int(z["alpha"][k]), int(z["seed"][k]))
        ids = z["ids"][z["ids_off"][k]:z["ids_off"][k + 1]]
        mate = z["mate"][z["mate_off"][k]:z["mate_off"][k + 1]]
        assert O.validate_matching_loop(n, eu, ev, ids, mate) == (bool(z["valid"][k]), bool(z["maximal"][k]))


@pytest.mark.parametrize("scale", [6, 10, 14])
def test_c_rmat_and_builder_match_numpy_restatements(scale):
    """lmxo_rmat_raw / lmxo_build_graph (the scale fixtures' generator) equal
    oracle.rmat_raw / build_graph_vec (pinned to the reference's numbering)."""
    u, v, w = O.rmat_raw(scale, 16, seed=3, permute=True)
    cu, cv, cw = O.c_rmat_raw(scale, 16, seed=3, permute=True)
    assert np.array_equal(u, cu) and np.array_equal(v, cv) and np.array_equal(w, cw)
    a = O.build_graph_vec(u, v, w, 1 << scale)
    b = O.c_build_graph(cu, cv, cw, 1 << scale)
    assert a[0] == b[0] and all(np.array_equal(x, y) for x, y in zip(a[1:], b[1:]))


def test_c_builder_matches_reference_numbering(golden_small):
    """lmxo_build_graph on the reference's raw lists (self-loops, duplicates,
    -0.0, ties): identical to the reference build_graph output."""
    for gi, n, raw, built, nv in small_cases(golden_small):
        u, v, w = (np.asarray(x) for x in raw)
        if u.size == 0:
            continue
        nn = n if n is not None else int(max(u.max(), v.max())) + 1
        _, eu, ev, ew = O.c_build_graph(u.astype(np.uint32), v.astype(np.uint32), w, nn)
        assert np.array_equal(eu, built[0]) and np.array_equal(ev, built[1]), gi
        assert np.array_equal(ew.view(np.uint64), np.asarray(built[2]).view(np.uint64)), gi


def test_scale_fixtures_are_consistent():
    """tests/golden/scale.json: every config the bench and GPU tests use, with
    the fields they compare; rgg22 and rmat24 were checked against the
    unmodified reference when they were made."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "scale.json")) as f:
        sc = json.load(f)
    for name in ("rgg22", "rmat24", "rmat26", "er24unit"):
        rec = sc[name]
        assert {"n", "m", "edges", "mate", "ids", "rounds", "weight", "matched"} <= set(rec)
        assert rec["rounds"][0][0] == rec["m"]
        assert sum(r[1] for r in rec["rounds"]) == rec["matched"]
        assert sum(r[2] for r in rec["rounds"]) == rec["m"]
    assert sc["rgg22"].get("reference_checked") and sc["rgg22"].get("generator_checked")
    assert sc["rmat24"].get("reference_checked") and sc["er24unit"].get("reference_checked")


def test_bsp_messages_match_reference():
    """oracle.bsp_messages vs the unmodified reference's bsp_local_max
    RoundMessages (tests/golden/bsp.npz, make_golden_bsp.py)."""
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "bsp.npz"))
    for k, (kind, size, alpha, seed, p, rr) in enumerate(z["cases"]):
        n, eu, ev, w = O.gen_random(int(size), int(alpha), int(seed)) if kind == 0 else O.gen_rgg(int(size), int(seed))
        want = [tuple(int(x) for x in r) for r in z["rows"][z["off"][k]:z["off"][k + 1]]]
        assert O.bsp_messages(n, eu, ev, w, int(p), int(seed), bool(rr)) == want
