#!/usr/bin/env python
"""bench.py -- input edges/s to a full local max maximal matching on B200.

Contract:
  python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference] [--workload rmat26]

One step = one full local max matching (all rounds, matchers.py:61-122 semantics)
of the workload graph, slot records resident in HBM when the timed region
starts.  value = m * K / T over the K timed steps (CUDA events on the
engine's stream, barrier + synchronize on both sides, max over ranks).
e2e = the same metric through the public API with pinned HOST buffers:
load_graph (H2D of edge_u/edge_v/edge_weight + device slot build) + match +
D2H of mate and matched ids, every step.

--impl reference times the reference's own CPU implementation of the path,
the unmodified locmax.local_max_seq (installed into baseline/_ref by
tools/install_reference.sh; the oracle's numpy port if it is absent), on a
bounded RMAT sample of the workload recipe, on rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (family, scale, edge factor).  rmat: Graph500 (a, b, c) = (.57, .19, .19),
    # U[0,1) weights, permuted labels.  er: uniform raw pairs (the C1 family,
    # BASELINE config C1 at 256x), unit weights.
    "rmat27": ("rmat", 27, 16),   # 2.1 G edges: the largest that one B200 holds (no golden; parity by oracle off-box)
    "rmat26": ("rmat", 26, 16), "rmat25": ("rmat", 25, 16), "rmat24": ("rmat", 24, 16),
    "rmat22": ("rmat", 22, 16), "rmat20": ("rmat", 20, 16), "rmat16": ("rmat", 16, 16),
    "er24unit": ("er", 24, 4), "er20unit": ("er", 20, 4),
    # rerandomize=False (the salts fixed for the run): the static (weight, salt)
    # layout serves unit weights on the scan loop (LMX_OPT_STATIC_ORDER)
    "er24unit-norr": ("er", 24, 4, False),
}


def wl(name: str):
    """(family, scale, edge factor, rerandomize) of a workload."""
    spec = WORKLOADS[name]
    return spec[0], spec[1], spec[2], (spec[3] if len(spec) > 3 else True)


def generate(eng, workload: str):
    fam, scale, ef, rr = wl(workload)
    if not rr:   # the layout for the fixed salts of the match seed
        eng.set_static_order(MATCH_SEED)
    if fam == "rmat":
        eng.gen_rmat(scale, ef, *RMAT_ABC, seed=GRAPH_SEED, permute=True)
        return f"RMAT scale {scale} edge factor {ef}"
    eng.gen_er(scale, ef, seed=GRAPH_SEED, unit=True)
    return f"random graph 2^{scale} vertices, {ef} * 2^{scale} uniform raw pairs, unit weights (C1 family)"
RMAT_ABC = (0.57, 0.19, 0.19)
GRAPH_SEED = 1
MATCH_SEED = 1
FALLBACK_HBM_GBS = 6650.0   # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json


def measured_hbm_gbs():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=5)
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sms.append(float(r[0]))
                mx = float(r[1])
            except ValueError:
                continue
            for nm, val in zip(names, r[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sms)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def rmat_floor_bytes(rounds):
    """B_floor = 32 (2S - m0), S = sum_r m_r (16-B slot records,
    every live slot read once and every surviving slot written once per round)."""
    S = sum(r.edges_before for r in rounds)
    m0 = rounds[0].edges_before if rounds else 0
    return 32 * (2 * S - m0), S, m0


def cpu_sample_graph(scale: int, family: str = "rmat", ef: int = 16):
    """A sample of the same recipe, generated on the host by the oracle's C
    restatement of the device generator + build_graph (test infrastructure,
    used here only to make the CPU arm's input)."""
    from oracle import oracle as O
    if family == "er":
        u, v, w = O.c_rmat_raw(scale, ef, 0.25, 0.25, 0.25, seed=GRAPH_SEED, permute=False)
        w[:] = 1.0
    else:
        u, v, w = O.c_rmat_raw(scale, ef, *RMAT_ABC, seed=GRAPH_SEED, permute=True)
    return O.c_build_graph(u, v, w, 1 << scale)


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def import_reference():
    """The UNMODIFIED reference package installed by tools/install_reference.sh
    into baseline/_ref (pip --target of /root/reference/pkg).  None if absent."""
    if os.path.isdir(os.path.join(REF_DIR, "locmax")) and REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import locmax.graph as lg
        import locmax.matchers as lm
    except ImportError:
        return None
    return lg, lm


def reference_graph(lg, n, eu, ev, w):
    """locmax.Graph from build_graph-ordered arrays: the CSR
    arrays as graph.py:108-115 lays them out; local_max_seq reads the edge arrays."""
    m = int(eu.size)
    sv = np.concatenate([eu, ev])
    se = np.concatenate([np.arange(m, dtype=np.int64), np.arange(m, dtype=np.int64)])
    order = np.argsort(sv * np.int64(max(m, 1)) + se, kind="stable")
    sv, se = sv[order], se[order]
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(sv, minlength=n), out=offsets[1:])
    arrs = [offsets, sv, se, np.ascontiguousarray(eu, dtype=np.int64), np.ascontiguousarray(ev, dtype=np.int64),
            np.ascontiguousarray(w, dtype=np.float64)]
    for a in arrs:
        a.setflags(write=False)
    return lg.Graph(int(n), *arrs)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    """--impl reference: the reference's own CPU implementation of the path,
    locmax.local_max_seq (matchers.py:61-122) from baseline/_ref, on a bounded
    RMAT sample of the workload recipe, rank 0 only.  If the reference is not
    installed, the oracle's numpy port of it (kind "port")."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    scale = args.cpu_sample_scale
    fam, _, ef, RR = wl(args.workload)
    n, eu, ev, w = cpu_sample_graph(scale, fam, ef)
    m = int(eu.size)
    ref = import_reference()
    if ref is not None:
        lg, lm = ref
        g = reference_graph(lg, n, eu, ev, w)
        run = lambda: lm.local_max_seq(g, MATCH_SEED, RR)   # noqa: E731
        kind, what = "reference", "locmax.local_max_seq (unmodified reference, baseline/_ref)"
    else:
        from oracle import oracle as O
        run = lambda: O.numpy_local_max(n, eu, ev, w, MATCH_SEED, RR)   # noqa: E731
        kind, what = "port", "oracle numpy port of local_max_seq (baseline/_ref not installed)"
    for _ in range(args.warmup):
        run()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        res = run()
        times.append(time.perf_counter() - t0)
    dt = sum(times)
    value = m * args.steps / dt
    rounds = len(res[1].rounds) if kind == "reference" else len(res.rounds)
    recipe = f"RMAT-{scale} ef{ef} (a,b,c)={RMAT_ABC} graph seed {GRAPH_SEED} permuted" if fam == "rmat" else \
        f"random graph 2^{scale}, {ef} * 2^{scale} uniform pairs, unit weights, graph seed {GRAPH_SEED}"
    sample = (f"{recipe}, n={n}, m={m}; "
              f"{args.steps} timed calls of {what}, match seed {MATCH_SEED}; 1 of {os.cpu_count()} host "
              f"cores ({cpu_model()}); the path is single-threaded numpy")
    line = {
        "impl": "reference", "metric": "input edges/s to full local max maximal matching",
        "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1000 / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": f"{fam}{scale}-sample-of-{args.workload}", "scale": scale,
                   "edge_factor": ef, "n": n, "m": m,
                   "rounds": rounds, "parallelism": "1 host core"},
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": 1, "kind": kind, "sample": sample,
                         "best_s": min(times), "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_leg(scale: int, reps: int = 3, family: str = "rmat", ef: int = 16, RR: bool = True):
    """The reference's local_max_seq (baseline/_ref; else the oracle's numpy
    port) on a bounded RMAT sample, best of `reps`, and the
    GPU result on the same sample checked identical to it."""
    from paper_1302_4587_b200 import Engine, Graph
    n, eu, ev, w = cpu_sample_graph(scale, family, ef)
    ref = import_reference()
    if ref is not None:
        lg, lm = ref
        g = reference_graph(lg, n, eu, ev, w)
        kind = "reference"
        run = lambda: lm.local_max_seq(g, MATCH_SEED, RR)   # noqa: E731
    else:
        from oracle import oracle as O
        kind = "port"
        run = lambda: O.numpy_local_max(n, eu, ev, w, MATCH_SEED, RR)   # noqa: E731
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        res = run()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    if kind == "reference":
        mm, tr = res
        ref_mate = np.asarray(mm.mate)
        ref_ids = np.array(sorted(mm.edges), dtype=np.int64)
        ref_rounds = [(r.edges_before, r.edges_matched, r.edges_removed) for r in tr.rounds]
    else:
        ref_mate, ref_ids, ref_rounds = res.mate, res.matched_ids, res.rounds
    with Engine(0) as eng:
        eng.load_graph(Graph(n, eu, ev, w))
        mate, ids, rounds = eng.match_raw(MATCH_SEED, RR)
    same = bool(np.array_equal(mate, ref_mate) and np.array_equal(ids, ref_ids)
                and [(r.edges_before, r.edges_matched, r.edges_removed) for r in rounds] == ref_rounds)
    what = "locmax.local_max_seq (unmodified reference, baseline/_ref)" if kind == "reference" else \
        "the oracle's numpy port of local_max_seq (baseline/_ref not installed)"
    return {
        "value": eu.size / best, "unit": "edges/s", "cores": 1, "kind": kind,
        "sample": (f"{family}-{scale} ef{ef} same recipe (n={n}, m={eu.size}); best of {reps} calls of {what}; "
                   f"1 of {os.cpu_count()} host cores used ({cpu_model()}); GPU result identical on this "
                   f"sample: {same}"),
        "best_s": best, "cpu_model": cpu_model(), "parity_on_sample": same,
    }


def load_traffic(workload: str):
    p = os.path.join(ROOT, "profiles", f"traffic_{workload}.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


def run_b200_dist(args):
    """N GPUs: the 1D-partitioned engine (paper_1302_4587_b200/dist.py) on the
    same workload graph, one partition per rank, NCCL exchanges per round.
    Strong scaling: the whole job is one matching of the workload graph."""
    import torch
    import torch.distributed as dist

    from paper_1302_4587_b200.dist import DistRank, TorchComm, run_rounds

    world, rank, local = dist_env()
    if args.backend != "nccl":   # test only: the ranks share the GPUs there are
        local %= max(torch.cuda.device_count(), 1)
    if "RANK" not in os.environ:   # --dist without torchrun: a one-rank group
        os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=os.environ.get("MASTER_PORT", "29531"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:   # test only: every rank on one GPU, host-staged collectives (no kernel waits on another rank)
        dist.init_process_group(args.backend)
    comm = TorchComm()
    comm.bind_device(dev)
    stream = torch.cuda.current_stream()
    fam, scale, ef, RR = wl(args.workload)
    if fam != "rmat":
        raise SystemExit("the partitioned bench runs the RMAT workloads")
    if world > 1:
        # the distributed builder: no rank ever holds the whole graph (config C5);
        # each rank keeps its local edges in page-locked host memory for the e2e leg
        from paper_1302_4587_b200.dist import build_rmat_distributed
        me = DistRank(None, world, rank, local, stream.cuda_stream, defer=True)
        build_rmat_distributed([me], comm, scale, ef, *RMAT_ABC, GRAPH_SEED, True, keep_records=not args.no_e2e)
    else:   # one rank (--dist): the whole graph; the single-GPU line carries the e2e number
        me = DistRank(None, world, rank, local, stream.cuda_stream,
                      rmat=dict(scale=scale, edge_factor=ef, a=RMAT_ABC[0], b=RMAT_ABC[1], c=RMAT_ABC[2],
                                seed=GRAPH_SEED, permute=True))
    n, m = me.n, me.m
    seeds = [MATCH_SEED + i for i in range(args.steps)]   # no two timed steps repeat a matching
    for i in range(args.warmup):
        run_rounds([me], comm, seeds[i % len(seeds)], True)
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    launches = 0
    for sd in seeds:
        run_rounds([me], comm, sd, True)
        launches += me.eng.last_timing()["round_launches"]
    ev1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = sampler.stop()
    rounds, records = run_rounds([me], comm, MATCH_SEED, True)   # untimed: the reported trace and counters
    tt = torch.tensor([ev0.elapsed_time(ev1)], device=dev, dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    T = float(tt.item())
    peak, _ = measured_hbm_gbs()
    ms_per_step = T / args.steps
    # per-rank algorithmic bytes from the rank's own device counters, summed
    by = scan_step_bytes(me.eng.last_round_counters(), me.n_local, me.m // world) if me.algo == "scan" else None
    tb = torch.tensor([float(by["probe"] + by["match"] + by["hist"]) if by else 0.0], device=dev,
                      dtype=torch.float64)
    dist.all_reduce(tb)
    step_bytes = float(tb.item())
    # ---- e2e at N GPUs: every step each rank copies its local edges (bsp.py:86-90,
    # with their global ids) from page-locked host memory, loads its partition
    # (K0), runs the matching protocol and reads its owned slice of mate back
    e2e = None
    if not args.no_e2e and world > 1:
        recs, k_local = me.host_records
        a, b = me.vertex_range(rank)
        hmate = torch.empty(max(b - a, 1), dtype=torch.int64, pin_memory=True)
        e2e_steps = max(1, min(args.steps, args.e2e_steps))

        def e2e_step():
            me.load_local_edges(recs, k_local, me.host_degrees, m)
            r_, _ = run_rounds([me], comm, MATCH_SEED, True)
            if b > a:
                hmate[: b - a].copy_(me.mate[a:b], non_blocking=True)
            return r_
        rounds_e = e2e_step()   # warm
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            rounds_e = e2e_step()
        torch.cuda.synchronize()
        te = torch.tensor([(time.perf_counter() - t0) * 1000.0, float(k_local) * 24.0 + float(n) * 4.0,
                           float(b - a) * 8.0],
                          device=dev, dtype=torch.float64)
        dist.all_reduce(te[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(te[1:])
        Te, h2d, d2h = (float(x) for x in te.tolist())
        assert rounds_e == rounds, "e2e matching trace differs from the timed one"
        e2e = {"value": m * e2e_steps / (Te / 1000.0), "unit": "edges/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": Te / e2e_steps, "steps": e2e_steps,
               "api": "DistRank.load_local_edges = lmx_dist_load_local (each rank's local edges with global "
                      "ids as 24-byte records + the global degrees u32[n], from page-locked host memory; the "
                      "partition's K0) + run_rounds + owned mate slice D2H; wall clock, max over ranks"}
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        # rank 0 alone, after the timed region: the reference on a bounded
        # sample of the same recipe (the other ranks wait at the barrier below)
        cpu = cpu_baseline_leg(args.cpu_baseline_scale, family=fam, ef=ef, RR=RR)
    if rank == 0:
        line = {
            "metric": "input edges/s to full local max maximal matching",
            "value": m * args.steps / (T / 1000.0), "unit": "edges/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": args.workload, "graph": f"RMAT scale {scale} edge factor {ef}",
                       "n": n, "m": m, "rounds": len(rounds), "parallelism": f"1d-vertex-partition{world}",
                       "build": "distributed (lmx_dist_rmat_*)" if world > 1 else "whole graph per rank",
                       "rank0_device_bytes": me.eng.device_bytes(),
                       "exchange_a_records": int(sum(records)),
                       "l2": "inputs larger than L2"},
            "roofline": {"bound": "hbm", "achieved": step_bytes / (ms_per_step / 1000.0) / 1e9 if step_bytes else None,
                         "peak": peak * world, "unit": "GB/s",
                         "frac": step_bytes / (ms_per_step / 1000.0) / 1e9 / (peak * world) if step_bytes else None,
                         "traffic": None,
                         "kernel": "whole step: the scan loop's algorithmic bytes (probe + match + histogram, "
                                   "DESIGN.md 4.3; histogram share taken as m/p) summed over ranks, against all ranks' HBM",
                         "algorithmic_bytes_per_step": step_bytes},
            "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clocks,
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()   # the other ranks wait for rank 0's CPU leg
    me.close()
    dist.destroy_process_group()
    return 0


def load_golden(workload: str):
    """Digests of the reference matching on this workload (tests/golden/scale.json,
    made by tests/golden/make_golden_scale.py from the pinned C oracle)."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "scale.json")) as f:
            return json.load(f).get(workload)
    except OSError:
        return None


def _sha(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).data).hexdigest()


def _edges_digest(eu, ev, w) -> str:
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(eu, dtype="<i8").data)
    h.update(np.ascontiguousarray(ev, dtype="<i8").data)
    h.update(np.ascontiguousarray(w, dtype="<f8").view("<u8").data)
    return h.hexdigest()[:32]


def parity_check(golden, g_host, mate_h, ids_h, rounds):
    """The timed workload's matching against the reference digests: graph
    (edge arrays), mate, matched ids, RoundStats, Matching.weight bits."""
    if golden is None:
        return {"checked": False, "why": "no golden digest for this workload"}
    weight = float(np.asarray(g_host.edge_weight)[ids_h].sum()) if ids_h.size else 0.0
    got = {
        "edges": _edges_digest(g_host.edge_u, g_host.edge_v, g_host.edge_weight),
        "mate": _sha(np.asarray(mate_h, dtype="<i8")), "ids": _sha(np.asarray(ids_h, dtype="<i8")),
        "rounds": [[r.edges_before, r.edges_matched, r.edges_removed] for r in rounds],
        "weight": weight.hex(),
    }
    fields = {k: got[k] == golden[k] for k in ("edges", "mate", "ids", "rounds", "weight")}
    return {"checked": True, "equal": all(fields.values()), "fields": fields,
            "oracle": "tests/golden/scale.json (pinned C oracle of matchers.py:61-122"
                      + (", = unmodified local_max_seq" if golden.get("reference_checked") else "") + ")",
            "matched": int(ids_h.size), "weight": weight}


def host_graph(eng, n, m):
    """The loaded graph as pinned host int64 / f64 arrays (a reference Graph)."""
    import torch
    from paper_1302_4587_b200 import Graph
    pu = torch.empty(m, dtype=torch.int64, pin_memory=True)
    pv = torch.empty(m, dtype=torch.int64, pin_memory=True)
    pw = torch.empty(m, dtype=torch.float64, pin_memory=True)
    g_dev = eng.export_graph()
    pu.numpy()[:] = g_dev.edge_u
    pv.numpy()[:] = g_dev.edge_v
    pw.numpy()[:] = g_dev.edge_weight
    del g_dev
    return Graph(n, pu.numpy(), pv.numpy(), pw.numpy()), pu, pv, pw


def property_check(eng, n, m, mate_h, ids_h, rounds):
    """No golden digest (a graph the oracle cannot hold here): the properties
    every local max matching has -- valid and maximal (validate_matching,
    graph.py:212-237, on the device), mate consistent with the ids, and a
    RoundStats trace that removes every edge (matchers.py:113-118)."""

    class _M:
        def __init__(self, mate, ids):
            self.mate, self._ids = mate, ids

        def sorted_edge_ids(self):
            return self._ids

    chk, weight = eng.validate(_M(np.asarray(mate_h), np.asarray(ids_h)))
    alive, trace_ok = m, True
    for r in rounds:
        trace_ok &= r.edges_before == alive and 0 < r.edges_matched <= r.edges_removed <= alive
        alive -= r.edges_removed
    fields = {"valid": bool(chk.valid), "maximal": bool(chk.maximal),
              "trace_removes_every_edge": bool(trace_ok and alive == 0),
              "matched_count": int(sum(r.edges_matched for r in rounds)) == int(np.asarray(ids_h).size),
              "mate_pairs": int((np.asarray(mate_h) >= 0).sum()) == 2 * int(np.asarray(ids_h).size)}
    return {"checked": True, "equal": None, "properties": fields, "all_properties": all(fields.values()),
            "why": "no golden digest for this workload (the C oracle needs more host memory than the build "
                   "container has): valid + maximal on the device, trace and mate consistency",
            "matched": int(np.asarray(ids_h).size), "weight": weight}


def scan_step_bytes(ctr, n, m):
    """Algorithmic bytes of one scan-loop matching per kernel,
    from the device counters of the step.
    probe: per listed vertex 8 B (list entry + 4-byte candidate word; round 0:
      the 8-byte first slot + the word write, 16 B), per slow-path vertex 20 B
      (ptr, segment bounds, word write), 8 B per slot read;
    match: per listed vertex 16 B (list entry, own and partner word, survivor
      append), per matched vertex 12 B (match round, mate);
    hist (pack + death-round histogram + matched-edge bits): 8 B per edge
      (lowpair) + 5 B per vertex (match round read, packed write) + n/8 (bitmap)
      + 32 B per matched edge (its candidate word, ptr, offset, slot, edge bit)."""
    A = [int(c[3]) for c in ctr]
    slow = [int(c[4]) for c in ctr]
    reads = [int(c[0]) for c in ctr]
    mv = [int(c[2]) for c in ctr]
    probe = sum(8 * a + 20 * s_ + 8 * r for a, s_, r in zip(A, slow, reads)) + (8 * A[0] if A else 0)
    match = sum(16 * a + 12 * v for a, v in zip(A, mv))
    hist = 8 * m + 5 * n + n // 8 + 32 * (sum(mv) // 2)
    return {"probe": probe, "match": match, "hist": hist, "launches": sum(1 for a in A if a > 0)}


def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_1302_4587_b200 import Engine, Graph

    world, rank, local = dist_env()
    if world > 1 or args.dist:
        return run_b200_dist(args)
    torch.cuda.set_device(local)
    stream = torch.cuda.current_stream()
    fam, scale, ef, RR = wl(args.workload)

    eng = Engine(local)
    eng.set_stream(stream.cuda_stream)
    graph_desc = generate(eng, args.workload)
    gen_setup_ms = eng.last_timing()["setup_ms"]
    n, m = eng.graph_size()

    # ---- K0 from device-resident edge arrays (the load the scan loop needs:
    # weight-ordered segments, candidates, lowpair), CUDA events on its stream
    load_ms = []
    load_note = None
    if m * 24 + 75 * m > 150e9:
        # the largest workloads (RMAT-27): the device edge inputs (24 B per
        # edge) and the load's peak (~75 B per edge) do not fit in HBM next to
        # each other; the generator's own load is the one that is matched
        load_note = ("device-input load not timed: %.0f GB of device inputs + ~%.0f GB load peak exceed HBM"
                     % (m * 24 / 1e9, m * 75 / 1e9))
    else:
        du, dv, dw = eng.export_graph_device()
        for rep in range(2):
            if rep == 1:
                eng.peak_device_bytes(reset=True)
            torch.cuda.synchronize()
            l0 = torch.cuda.Event(enable_timing=True)
            l1 = torch.cuda.Event(enable_timing=True)
            l0.record(stream)
            eng.load_graph_device(n, du, dv, dw)
            l1.record(stream)
            torch.cuda.synchronize()
            load_ms.append(l0.elapsed_time(l1))
        del du, dv, dw
    device_memory = {"after_load_GB": round(eng.device_bytes() / 1e9, 2),
                     "load_peak_GB": round(eng.peak_device_bytes() / 1e9, 2),
                     "note": "engine allocations (device edge inputs of the load excluded)"}
    torch.cuda.empty_cache()
    load_device_ms = min(load_ms) if load_ms else None

    mate = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    ids = torch.empty(max(n // 2 + 1, 1), dtype=torch.int64, device="cuda")

    # every timed step matches with its own seed (MATCH_SEED + i): no two
    # steps repeat a matching.  A static-order load serves its one seed only.
    seeds = [MATCH_SEED if eng.static_order() else MATCH_SEED + i for i in range(args.steps)]
    for i in range(args.warmup):
        eng.match_device(seeds[i % len(seeds)], mate, ids, RR)

    # ---- timed region: K full matchings from HBM-resident slots
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    launches = 0
    rounds_exec = 0
    for sd in seeds:
        eng.match_device(sd, mate, ids, RR)
        t = eng.last_timing()
        launches += t["round_launches"]
        rounds_exec += t["rounds_executed"]
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    T = ev0.elapsed_time(ev1)

    # ---- per-kernel CUDA-event timeline of the same matchings (after the
    # timed region: its per-launch events would perturb the headline)
    eng.set_kernel_timing(True)
    rk_ms = mk_ms = hk_ms = 0.0
    for sd in seeds:
        eng.match_device(sd, mate, ids, RR)
        t = eng.last_timing()
        rk_ms += t["round_kernel_ms"]
        mk_ms += t["match_kernel_ms"]
        hk_ms += t["hist_kernel_ms"]
    eng.set_kernel_timing(False)
    rk_ms, mk_ms, hk_ms = rk_ms / args.steps, mk_ms / args.steps, hk_ms / args.steps

    # ---- the golden seed's matching (untimed) for the parity digests; its
    # device counters give the algorithmic bytes below
    nm = eng.match_device(MATCH_SEED, mate, ids, RR)
    rounds = eng.last_rounds()
    mate_h = mate[:n].cpu().numpy()
    ids_h = ids[:nm].cpu().numpy()
    n_matched = int(sum(r.edges_matched for r in rounds))

    ms_per_step = T / args.steps
    value = m * args.steps / (T / 1000.0)
    peak, peak_src = measured_hbm_gbs()
    src = "measured (MEASURED_PEAKS.json hbm_gbs)" if peak_src == "measured" else \
        "fallback 6.65 TB/s (B200_PROFILING.md)"
    algo = eng.algo()
    traffic = load_traffic(args.workload)
    if algo == "scan":
        by = scan_step_bytes(eng.last_round_counters(), n, m)
        if traffic and traffic.get("kernel") != "lmx_scan_loop_kernel":
            traffic = None
        # the dominant kernel: the persistent round loop (all probes + matches of
        # one matching in ONE launch); its duration = the sum of the per-phase
        # globaltimer stamps (probe + match) of the same launches
        loop_ms = rk_ms + mk_ms
        loop_bytes = by["probe"] + by["match"]
        loop_gbs = loop_bytes / (loop_ms / 1000.0) / 1e9 if loop_ms > 0 else None
        roofline = {
            "bound": "hbm", "achieved": loop_gbs, "peak": peak, "unit": "GB/s",
            "frac": loop_gbs / peak if loop_gbs else None,
            "traffic": traffic.get("bytes_per_launch") if traffic else None,
            "kernel": "lmx_scan_loop_kernel (the whole round loop of one matching: candidate probes + "
                      "mutual checks, one cooperative launch)",
            "algorithmic_bytes_per_step": loop_bytes,
            "algorithmic_bytes_per_launch": loop_bytes,
            "kernel_ms_per_step": loop_ms, "peak_source": src,
            "traffic_source": traffic.get("source") if traffic else None,
            "traffic_over_algorithmic": (traffic["bytes_per_launch"] / loop_bytes) if traffic else None,
        }
        kern = {"probe": (by["probe"], rk_ms), "match": (by["match"], mk_ms), "hist+edge_bits": (by["hist"], hk_ms)}
        step_bytes = by["probe"] + by["match"] + by["hist"]
    else:
        # compacting loop, 8-byte slots {nbr, id} (UNIFORM / DISTINCT layouts):
        # every live slot read once and every surviving slot written once per
        # round, 16 (m_r + m_{r+1}) bytes; the match kernel 16 B per listed
        # vertex (list, own and partner candidate, survivor append) + 12 B per
        # matched vertex, listed vertices ~ live vertices <= live slots
        S = sum(r.edges_before for r in rounds)
        m0 = rounds[0].edges_before if rounds else 0
        B_round = 16 * (2 * S - m0)
        ctr = eng.last_round_counters()
        listed = int(sum(int(sum(c[3:8])) for c in ctr))
        mv = int(sum(int(c[2]) for c in ctr))
        B_match = 16 * listed + 12 * mv
        gbs = B_round / (rk_ms / 1000.0) / 1e9 if rk_ms > 0 else None
        roofline = {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                    "frac": gbs / peak if gbs else None,
                    "traffic": traffic.get("bytes_per_launch") if traffic and traffic.get("kernel") ==
                    "lmx_round_kernel" else None,
                    "kernel": "lmx_round_kernel (fused kill+compact+argmax, all rounds; 8-byte slots)",
                    "algorithmic_bytes_per_step": B_round, "kernel_ms_per_step": rk_ms, "peak_source": src,
                    "byte_model": "16 (2 S - m0), S = sum_r m_r: each live slot (8 B) read, each survivor written"}
        kern = {"round": (B_round, rk_ms), "match": (B_match, mk_ms)}
        step_bytes = B_round + B_match
    step_gbs = step_bytes / (ms_per_step / 1000.0) / 1e9
    step_roofline = {
        "achieved": step_gbs, "peak": peak, "unit": "GB/s", "frac": step_gbs / peak,
        "algorithmic_bytes_per_step": step_bytes, "ms_per_step": ms_per_step,
        "definition": "sum of the step's kernels' algorithmic bytes (scan loop: probe + match + death-round "
                      "histogram + matched-edge bits, DESIGN.md 4.3) / device step time / measured peak",
        "kernels": {k: {"algorithmic_bytes": b, "ms": t_, "gbs": (b / (t_ / 1000.0) / 1e9) if t_ > 0 else None}
                    for k, (b, t_) in kern.items()},
    }

    # ---- parity: digests against the golden, or (no golden: the largest
    # workloads) the size-independent properties on the device
    golden = load_golden(args.workload)
    need_host = golden is not None or (not args.no_e2e and load_note is None)
    hg = pu = pv = pw = None
    if need_host:   # host copy of the graph: parity digests and the e2e leg's pinned inputs
        hg, pu, pv, pw = host_graph(eng, n, m)
    if args.no_parity:
        parity = {"checked": False, "why": "--no-parity"}
    elif golden is not None:
        parity = parity_check(golden, hg, mate_h, ids_h, rounds)
    else:
        parity = property_check(eng, n, m, mate_h, ids_h, rounds)

    # ---- e2e: public API with pinned host buffers, H2D + device build + match + D2H every step
    e2e = None
    if not args.no_e2e and load_note is not None:
        e2e = {"unavailable": "the device-input load did not fit (see load_device_note)"}
    elif not args.no_e2e:
        eng.set_relabel(args.e2e_relabel)
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        # warm: two steps, so the pinned output pool holds the buffers of the
        # result a caller keeps while the next step allocates (steady state)
        keep = None
        for _ in range(2):
            eng.load_graph(hg)
            keep = eng.match_raw(MATCH_SEED, RR)
        del keep
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            eng.load_graph(hg)
            hmate, hids, hrounds = eng.match_raw(MATCH_SEED, RR)
        e1.record(stream)
        torch.cuda.synchronize()
        Te = max(e0.elapsed_time(e1), (time.perf_counter() - t0) * 1000.0)
        assert hrounds == rounds and np.array_equal(hids, ids_h) and np.array_equal(hmate, mate_h)
        e2e = {"value": m * e2e_steps / (Te / 1000.0), "unit": "edges/s",
               "h2d_bytes_per_step": int(m * 16), "d2h_bytes_per_step": int(n * 8 + n_matched * 8),
               "h2d_note": "host arrays read: m*24 B (int64 u, v, f64 w); crossing the link: m*16 B -- the "
                           "endpoints are range-checked and narrowed to u32 by host threads into a pinned "
                           "staging ring (csrc/lmx_hostload.cpp, lmx_setup.cu load_host_narrowed)",
               "ms_per_step": Te / e2e_steps, "steps": e2e_steps,
               "setup_ms_last": eng.last_timing()["setup_ms"],
               "api": "Engine.load_graph(Graph of pinned host arrays) + Engine.match_raw (lmx_load_graph + "
                      "lmx_match, host outputs)",
               "relabel": args.e2e_relabel}
    del hg, pu, pv, pw

    cpu = None
    if not args.no_cpu_baseline:
        eng.close()
        cpu = cpu_baseline_leg(args.cpu_baseline_scale, family=fam, ef=ef, RR=RR)

    line = {
        "metric": "input edges/s to full local max maximal matching", "value": value,
        "unit": "edges/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": args.workload, "graph": graph_desc,
                   "rmat_abc": list(RMAT_ABC) if fam == "rmat" else [0.25, 0.25, 0.25],
                   "graph_seed": GRAPH_SEED, "match_seed": MATCH_SEED,
                   "timed_seeds": f"{seeds[0]}..{seeds[-1]}" if len(set(seeds)) > 1 else seeds[0],
                   "rerandomize": RR,
                   "static_order": eng.static_order(),
                   "permuted_labels": fam == "rmat", "n": n, "m": m, "rounds": len(rounds),
                   "matched_edges": n_matched, "round_loop": algo, "parallelism": "dp1",
                   "l2": "inputs larger than L2 (slot records %.1f GB >> 126 MB)" % (2 * m * 8 / 1e9)},
        "parity": parity,
        "load_device_ms": load_device_ms,
        "load_device_note": load_note or
                            "lmx_load_graph from device-resident int64/f64 edge arrays (validation, narrowing, "
                            "degrees, relabelling, weight-ordered segments, candidates, lowpair), CUDA events, "
                            "best of 2; not inside `value`",
        "value_with_load": m / ((load_device_ms + ms_per_step) / 1000.0) if load_device_ms else None,
        "device_memory": device_memory,
        "roofline": roofline, "step_roofline": step_roofline,
        "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
        "gpu_launches": launches, "rounds_enqueued": rounds_exec,
        "generator_setup_ms": gen_setup_ms,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="rmat26")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-sample-scale", type=int, default=20,
                    help="RMAT scale of the reference arm's per-step sample")
    ap.add_argument("--cpu-baseline-scale", type=int, default=21,
                    help="RMAT scale of the cpu_baseline leg (best of 3)")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--backend", default="nccl", help=argparse.SUPPRESS)
    ap.add_argument("--e2e-relabel", default="once", choices=("auto", "on", "off", "once"),
                    help="degree relabelling of the e2e leg's loads (Engine.set_relabel); each e2e step is "
                         "one load + one matching: 'once', the one-shot entry points' choice")
    ap.add_argument("--dist", action="store_true",
                    help="use the 1D-partitioned multi-GPU engine even at one rank (NCCL code path check)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
