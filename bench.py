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

--impl reference times the reference algorithm's CPU implementation (the
oracle's numpy port of local_max_seq, same whole-array numpy operations as
matchers.py:87-119, single-threaded like the reference) on a bounded sample
of the same workload family, on rank 0 only.
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
    # name: RMAT scale, edge factor; Graph500 (a, b, c) = (.57, .19, .19), U[0,1) weights
    "rmat26": 26, "rmat25": 25, "rmat24": 24, "rmat22": 22, "rmat20": 20, "rmat16": 16,
}
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


def cpu_sample_graph(scale: int):
    """RMAT sample of the same recipe, generated on the CPU by the oracle's restatement."""
    from oracle import oracle as O
    u, v, w = O.rmat_raw(scale, 16, *RMAT_ABC, seed=GRAPH_SEED, permute=True)
    return O.build_graph_vec(u, v, w, 1 << scale)


def run_reference(args):
    """--impl reference: the reference algorithm (numpy port, 1 core) on a bounded sample."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O
    scale = args.cpu_sample_scale
    n, eu, ev, w = cpu_sample_graph(scale)
    m = int(eu.size)
    for _ in range(args.warmup):
        O.numpy_local_max(n, eu, ev, w, MATCH_SEED, True)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        res = O.numpy_local_max(n, eu, ev, w, MATCH_SEED, True)
    dt = time.perf_counter() - t0
    value = m * args.steps / dt
    sample = (f"RMAT-{scale} ef16 (a,b,c)={RMAT_ABC} seed {GRAPH_SEED} permuted, m={m}, "
              f"{args.steps} timed runs of numpy_local_max (matchers.py:61-122 numpy ops)")
    line = {
        "impl": "reference", "metric": "input edges/s to full local max maximal matching",
        "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1000 / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": f"rmat{scale}-sample-of-{args.workload}", "scale": scale,
                   "edge_factor": 16, "rmat_abc": list(RMAT_ABC), "n": n, "m": m,
                   "rounds": len(res.rounds), "parallelism": "1 host core"},
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": 1, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_leg(eng_sample_scale: int):
    """Time the oracle's numpy port (the reference's algorithm, 1 core) on a
    bounded RMAT sample and check the GPU gives the identical matching on it."""
    from oracle import oracle as O
    from paper_1302_4587_b200 import Engine, Graph
    n, eu, ev, w = cpu_sample_graph(eng_sample_scale)
    t0 = time.perf_counter()
    res = O.numpy_local_max(n, eu, ev, w, MATCH_SEED, True)
    dt = time.perf_counter() - t0
    with Engine(0) as eng:
        g = Graph(n, eu, ev, w)
        eng.load_graph(g)
        mate, ids, rounds = eng.match_raw(MATCH_SEED, True)
    same = bool(np.array_equal(mate, res.mate) and np.array_equal(ids, res.matched_ids)
                and [(r.edges_before, r.edges_matched, r.edges_removed) for r in rounds] == res.rounds)
    return {
        "value": eu.size / dt, "unit": "edges/s", "cores": 1, "kind": "port",
        "sample": (f"RMAT-{eng_sample_scale} ef16 same recipe (m={eu.size}), one run of the oracle's "
                   f"numpy port of local_max_seq (matchers.py:61-122 ops) on {os.cpu_count()} host cores "
                   f"(1 used); GPU result identical on this sample: {same}"),
        "parity_on_sample": same,
    }


def step_roofline(algo, ctr, probe_ms, match_ms, hist_ms, ms_per_step, n, m, n_rounds, B_floor, peak, peak_src,
                  traffic):
    """Roofline of the dominant kernel.  Scan loop: the
    candidate-probe kernel (largest share of the step), with its algorithmic
    bytes from the device counters of the step: per probed vertex 8 B (list
    entry + 4-byte candidate word; round 0 reads the 8-byte first slot and
    writes the word: 16 B), per slow-path vertex 20 B (ptr, degree, offset,
    word write), 8 B per slot read.  Match kernel: 16 B per listed vertex (list
    entry, own and partner words, survivor append) + 12 B per matched vertex
    (match round, mate).  Histogram pass: 8 B per edge + 5 B per vertex, plus
    the matched-edge bit pass (bitmap, and per matched lower endpoint word,
    ptr, offset, slot, edge id, bit: 32 B).
    Compacting loop: SURVEY.md §8d's B_floor over the round kernel."""
    src = "measured (MEASURED_PEAKS.json hbm_gbs)" if peak_src == "measured" else \
        "fallback 6.65 TB/s (B200_PROFILING.md)"
    want = "lmx_scan_round_kernel" if algo == "scan" else "lmx_round_kernel"
    if traffic and traffic.get("kernel") != want:
        traffic = None   # a capture of another kernel
    if algo == "scan":
        A = [int(c[3]) for c in ctr]
        slow = [int(c[4]) for c in ctr]
        reads = [int(c[0]) for c in ctr]
        mv = [int(c[2]) for c in ctr]
        probe_bytes = sum(8 * a + 20 * s + 8 * r for a, s, r in zip(A, slow, reads)) + (8 * A[0] if A else 0)
        launches = sum(1 for a in A if a > 0)
        match_bytes = sum(16 * a + 12 * v for a, v in zip(A, mv))
        hist_bytes = 8 * m + 5 * n + n // 8 + 32 * (sum(mv) // 2)
        achieved = probe_bytes / (probe_ms / 1000.0) / 1e9 if probe_ms > 0 else None
        return {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak if achieved else None,
            "traffic": traffic.get("bytes_per_launch") if traffic else None,
            "kernel": "lmx_scan_round_kernel (candidate probes, all rounds)",
            "algorithmic_bytes_per_step": probe_bytes,
            "algorithmic_bytes_per_launch": probe_bytes / max(launches, 1),
            "kernel_ms_per_step": probe_ms, "peak_source": src,
            "traffic_source": traffic.get("source") if traffic else None,
            # The probe's useful bytes are gathered 4-8 B at a time from scattered
            # vertices; a DRAM sector is 32 B.  The measured DRAM traffic over the
            # kernel time is the bandwidth the access pattern actually draws.
            "measured_traffic_gbs": (traffic["bytes_per_launch"] * launches / (probe_ms / 1000.0) / 1e9)
            if traffic and probe_ms > 0 else None,
            "other_kernels": {
                "lmx_scan_match_kernel": {"ms_per_step": match_ms, "algorithmic_bytes": match_bytes,
                                          "achieved_gbs": match_bytes / (match_ms / 1000.0) / 1e9
                                          if match_ms > 0 else None},
                "lmx_scan_hist_hub_kernel (+ pack, + lmx_scan_edge_bits)": {
                    "ms_per_step": hist_ms, "algorithmic_bytes": hist_bytes,
                                                  "achieved_gbs": hist_bytes / (hist_ms / 1000.0) / 1e9
                                                  if hist_ms > 0 else None},
            },
            "compacting_floor": {
                "bytes": B_floor, "ms_at_peak": B_floor / (peak * 1e9) * 1000.0,
                "note": "SURVEY.md 8d floor of the per-round compacting algorithm (every live slot read and "
                        "every survivor written each round); the weight-ordered scan moves less than this, so "
                        "the step can finish below ms_at_peak"},
        }
    achieved = B_floor / (probe_ms / 1000.0) / 1e9 if probe_ms > 0 else None
    return {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak if achieved else None,
        "traffic": traffic.get("bytes_per_launch") if traffic else None,
        "kernel": "lmx_round_kernel (fused kill+compact+argmax, all rounds)",
        "algorithmic_bytes_per_step": B_floor, "algorithmic_bytes_per_launch": B_floor / max(n_rounds, 1),
        "kernel_ms_per_step": probe_ms, "match_kernel_ms_per_step": match_ms,
        "step_frac": (B_floor / (ms_per_step / 1000.0) / 1e9) / peak, "peak_source": src,
        "traffic_source": traffic.get("source") if traffic else None,
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
    if "RANK" not in os.environ:   # --dist without torchrun: a one-rank group
        os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=os.environ.get("MASTER_PORT", "29531"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    comm = TorchComm()
    comm.bind_device(dev)
    stream = torch.cuda.current_stream()
    scale = WORKLOADS[args.workload]
    me = DistRank(None, world, rank, local, stream.cuda_stream,
                  rmat=dict(scale=scale, edge_factor=16, a=RMAT_ABC[0], b=RMAT_ABC[1], c=RMAT_ABC[2],
                            seed=GRAPH_SEED, permute=True))
    n, m = me.n, me.m
    for _ in range(args.warmup):
        rounds, _ = run_rounds([me], comm, MATCH_SEED, True)
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    launches = 0
    for _ in range(args.steps):
        rounds, records = run_rounds([me], comm, MATCH_SEED, True)
        launches += me.eng.last_timing()["round_launches"]
    ev1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = sampler.stop()
    tt = torch.tensor([ev0.elapsed_time(ev1)], device=dev, dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    T = float(tt.item())
    B_floor, S, m0 = rmat_floor_bytes(rounds)
    peak, _ = measured_hbm_gbs()
    ms_per_step = T / args.steps
    if rank == 0:
        line = {
            "metric": "input edges/s to full local max maximal matching",
            "value": m * args.steps / (T / 1000.0), "unit": "edges/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": args.workload, "graph": f"RMAT scale {scale} edge factor 16",
                       "n": n, "m": m, "rounds": len(rounds), "parallelism": f"1d-vertex-partition{world}",
                       "exchange_a_records": int(sum(records)),
                       "l2": "inputs larger than L2"},
            "roofline": {"bound": "hbm", "achieved": B_floor / (ms_per_step / 1000.0) / 1e9,
                         "peak": peak * world, "unit": "GB/s",
                         "frac": B_floor / (ms_per_step / 1000.0) / 1e9 / (peak * world),
                         "traffic": None,
                         "kernel": "whole step against SURVEY.md 8d's compacting floor B_floor (all ranks' HBM)",
                         "algorithmic_bytes_per_step": B_floor},
            "cpu_baseline": None, "e2e": None,
            "e2e_note": "not measured on the partitioned path: every rank would need the full 25 GB host graph "
                        "pinned; the one-GPU line carries the end-to-end number",
            "clocks": clocks,
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    me.close()
    dist.destroy_process_group()
    return 0


def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_1302_4587_b200 import Engine, Graph

    world, rank, local = dist_env()
    if world > 1 or args.dist:
        return run_b200_dist(args)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    scale = WORKLOADS[args.workload]

    eng = Engine(local)
    eng.set_stream(stream.cuda_stream)
    eng.gen_rmat(scale, 16, *RMAT_ABC, seed=GRAPH_SEED, permute=True)
    setup_ms = eng.last_timing()["setup_ms"]
    n, m = eng.graph_size()
    mate = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    ids = torch.empty(max(n // 2 + 1, 1), dtype=torch.int64, device="cuda")

    for _ in range(args.warmup):
        eng.match_device(MATCH_SEED, mate, ids)
    rounds = eng.last_rounds()

    # ---- timed region: K full matchings from HBM-resident slots
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    launches = 0
    rounds_exec = 0
    for _ in range(args.steps):
        eng.match_device(MATCH_SEED, mate, ids)
        t = eng.last_timing()
        launches += t["round_launches"]
        rounds_exec += t["rounds_executed"]
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    T = ev0.elapsed_time(ev1)
    if world > 1:
        tt = torch.tensor([T], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        T = float(tt.item())
    assert eng.last_rounds() == rounds, "matching trace changed between steps"

    # ---- per-kernel CUDA-event timeline of the same matchings (after the
    # timed region: its per-launch events would perturb the headline)
    eng.set_kernel_timing(True)
    rk_ms = mk_ms = hk_ms = 0.0
    for _ in range(args.steps):
        eng.match_device(MATCH_SEED, mate, ids)
        t = eng.last_timing()
        rk_ms += t["round_kernel_ms"]
        mk_ms += t["match_kernel_ms"]
        hk_ms += t["hist_kernel_ms"]
    eng.set_kernel_timing(False)
    assert eng.last_rounds() == rounds, "matching trace changed between steps"
    n_matched = int(sum(r.edges_matched for r in rounds))

    B_floor, S, m0 = rmat_floor_bytes(rounds)
    assert m0 == m
    ms_per_step = T / args.steps
    value = world * m * args.steps / (T / 1000.0)
    peak, peak_src = measured_hbm_gbs()
    algo = eng.algo()
    roofline = step_roofline(algo, eng.last_round_counters(), rk_ms / args.steps, mk_ms / args.steps,
                             hk_ms / args.steps, ms_per_step, n, m, len(rounds), B_floor, peak, peak_src,
                             load_traffic(args.workload))

    # ---- e2e: public API with pinned host buffers, H2D + device build + match + D2H every step
    e2e = None
    if not args.no_e2e:
        g_dev = eng.export_graph()   # host copy of the workload graph
        pu = torch.empty(m, dtype=torch.int64, pin_memory=True)
        pv = torch.empty(m, dtype=torch.int64, pin_memory=True)
        pw = torch.empty(m, dtype=torch.float64, pin_memory=True)
        pu.numpy()[:] = g_dev.edge_u
        pv.numpy()[:] = g_dev.edge_v
        pw.numpy()[:] = g_dev.edge_weight
        del g_dev
        hg = Graph(n, pu.numpy(), pv.numpy(), pw.numpy())
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        # warm: two steps, so the pinned output pool holds the buffers of the
        # result a caller keeps while the next step allocates (steady state)
        keep = None
        for _ in range(2):
            eng.load_graph(hg)
            keep = eng.match_raw(MATCH_SEED, True)
        del keep
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            eng.load_graph(hg)
            hmate, hids, hrounds = eng.match_raw(MATCH_SEED, True)
        e1.record(stream)
        torch.cuda.synchronize()
        Te = max(e0.elapsed_time(e1), (time.perf_counter() - t0) * 1000.0)
        if world > 1:
            tt = torch.tensor([Te], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            Te = float(tt.item())
        assert hrounds == rounds and hids.size == n_matched
        e2e = {"value": world * m * e2e_steps / (Te / 1000.0), "unit": "edges/s",
               "h2d_bytes_per_step": int(m * 24), "d2h_bytes_per_step": int(n * 8 + n_matched * 8),
               "ms_per_step": Te / e2e_steps, "steps": e2e_steps,
               "setup_ms_last": eng.last_timing()["setup_ms"]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        eng.close()
        cpu = cpu_baseline_leg(args.cpu_sample_scale)

    if rank == 0:
        line = {
            "metric": "input edges/s to full local max maximal matching", "value": value,
            "unit": "edges/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": args.workload, "graph": f"RMAT scale {scale} edge factor 16",
                       "rmat_abc": list(RMAT_ABC), "graph_seed": GRAPH_SEED, "match_seed": MATCH_SEED,
                       "permuted_labels": True, "n": n, "m": m, "rounds": len(rounds),
                       "matched_edges": n_matched, "S_over_m0": S / m0, "round_loop": algo,
                       "parallelism": "dp1" if world == 1 else f"replicas{world}",
                       "l2": "inputs larger than L2 (slot records %.1f GB >> 126 MB)" % (2 * m * 12 / 1e9),
                       "setup_ms": setup_ms},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches, "rounds_enqueued": rounds_exec,
            # BASELINE north_star target: >= 50 % of HBM-roofline edges/s, the roofline being
            # SURVEY 8d's floor of the matching (B_floor bytes at the measured peak bandwidth)
            "north_star": {
                "target_frac": 0.5,
                "roofline_edges_per_s": m / (B_floor / (peak * 1e9)),
                "achieved_frac": value / world / (m / (B_floor / (peak * 1e9))),
                "roofline_definition": "m / (B_floor / peak), B_floor = 32 (2S - m0) bytes (SURVEY.md 8d)",
            },
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="rmat26")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-sample-scale", type=int, default=20)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="use the 1D-partitioned multi-GPU engine even at one rank (NCCL code path check)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
