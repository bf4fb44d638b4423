"""Run every BASELINE.json config through the B200 engine: device time per
matching, round loop used, and parity with the oracle where the CPU side
finishes in seconds.  Writes one JSON object (profiles/r1_configs.json).

C1 ER n=2^16 avg degree 8, unit weights   -> parity vs oracle (C restatement)
C2 RGG n=2^22, Euclidean weights          -> parity vs oracle (C restatement)
C3 RMAT-24 ef16, random weights           -> device timing, validate on GPU
C4 mesh 2^24 coarsening                   -> levels, end-to-end time
(N* RMAT-26 is bench.py's workload; C5 RMAT-28 needs 8 GPUs.)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1302_4587_b200 import Engine, Graph  # noqa: E402
from paper_1302_4587_b200.coarsen import coarsen_mesh  # noqa: E402


def timed_match(eng, g, seed, reps=5):
    best = None
    for _ in range(reps):
        m, tr = eng.match(g, seed, True)
        best = tr.device_millis if best is None else min(best, tr.device_millis)
    return m, tr, best


def main():
    out = {}
    eng = Engine(0)
    # C1
    n, eu, ev, w = O.gen_random(1 << 16, 4, 1, unit=True)
    g = Graph(n, eu, ev, w)
    eng.load_graph(g)
    m, tr, ms = timed_match(eng, g, 1)
    ref = O.c_local_max(n, eu, ev, w, 1, True)
    out["C1_er16_unit"] = {"n": n, "m": int(eu.size), "layout": eng.layout(), "round_loop": eng.algo(),
                           "rounds": len(tr.rounds), "device_ms": ms,
                           "parity": bool(np.array_equal(np.asarray(m.mate), ref.mate))}
    print(out["C1_er16_unit"], flush=True)
    # C2
    t = time.perf_counter()
    n, eu, ev, w = O.gen_rgg(22, 1)
    gen_s = time.perf_counter() - t
    g = Graph(n, eu, ev, w)
    eng.load_graph(g)
    setup = eng.last_timing()["setup_ms"]
    m, tr, ms = timed_match(eng, g, 1)
    t = time.perf_counter()
    ref = O.c_local_max(n, eu, ev, w, 1, True)
    cpu_s = time.perf_counter() - t
    out["C2_rgg22"] = {"n": n, "m": int(eu.size), "layout": eng.layout(), "round_loop": eng.algo(),
                       "rounds": len(tr.rounds), "device_ms": ms, "setup_ms": setup,
                       "edges_per_s": eu.size / (ms / 1e3), "host_generation_s": gen_s,
                       "oracle_c_s": cpu_s, "parity": bool(np.array_equal(np.asarray(m.mate), ref.mate)) and
                       [(r.edges_before, r.edges_matched, r.edges_removed) for r in tr.rounds] == ref.rounds}
    print(out["C2_rgg22"], flush=True)
    # C3
    eng.gen_rmat(24, 16, 0.57, 0.19, 0.19, seed=1, permute=True)
    gr = eng.export_graph()
    m, tr, ms = timed_match(eng, gr, 1)
    chk, weight = eng.validate(m)
    out["C3_rmat24"] = {"n": gr.num_vertices, "m": int(np.asarray(gr.edge_u).size), "layout": eng.layout(),
                        "round_loop": eng.algo(), "relabeled": eng.relabeled(), "rounds": len(tr.rounds),
                        "device_ms": ms, "edges_per_s": np.asarray(gr.edge_u).size / (ms / 1e3),
                        "valid": chk.valid, "maximal": chk.maximal, "weight": weight}
    print(out["C3_rmat24"], flush=True)
    del gr
    eng.close()
    # C4
    levels, final, total_ms = coarsen_mesh(4096, 0)
    out["C4_mesh4096_coarsening"] = {
        "levels": len(levels), "final": list(final), "end_to_end_ms": total_ms,
        "level0": {"n": levels[0].n, "m": levels[0].m, "matched": levels[0].matched,
                   "rounds": len(levels[0].rounds), "match_ms": levels[0].match_ms},
        "match_ms_all_levels": sum(lv.match_ms for lv in levels)}
    print(out["C4_mesh4096_coarsening"], flush=True)
    path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/configs.json"
    with open(path, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
