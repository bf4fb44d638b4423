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
