"""1D-partitioned local max over several GPUs (row (e) of SURVEY.md §8).

Mirrors ``locmax.bsp.bsp_local_max(g, p, seed, rerandomize)``
(``/root/reference/pkg/src/locmax/bsp.py:101-205``).  The reference
simulates p workers in one process; here each worker is a liblmx context:
* it owns one of p contiguous vertex ranges with equal degree sums, cut
  exactly as ``partition_graph`` cuts them (``bsp.py:60-98``);
* it holds the slots of every edge incident to its range.

Each round is driven by the host over a communicator:

1. ``lmx_dist_round``: owned vertices raise candidates (superstep 1,
   ``bsp.py:139-146``).
2. Exchange A (barrier 1, ``bsp.py:148-167``): for every owned live vertex
   whose candidate partner is remote, one record ``{partner, edge id}`` goes
   to the partner's owner.  This is an all-to-all-v.  A vertex is matched
   across the cut iff its owner *receives* the record of its own candidate
   edge.
3. ``lmx_dist_match``: local plus confirmed cross-rank matches; mate, matched
   edges, and the next round's lists.
4. Exchange B (barrier 2, ``bsp.py:169-170``): the owned words of the
   matched bitmap are all-gathered.  Every rank then filters dead slots in
   the next round.
5. An all-reduce of (live slots, matched vertices) gives ``RoundStats`` and
   termination.

The matching equals the single-GPU one for every p, as ``bsp.py:113-115``
promises.

Communicators:

* ``LocalComm``: p contexts in one process on one GPU, exchanging through
  device copies.  This is the reference's own "logical workers" mode
  (``bsp.py:13-16``).  It drives ``run_matcher(..., engine="b200-dist")``.
  It also runs the multi-rank kernels on one GPU, sequentially and with no
  kernel waiting on another.
* ``TorchComm``: one process per GPU under ``torch.distributed`` (NCCL over
  NVLink / NVSwitch; ``gloo`` works too), launched by torchrun.
"""

from __future__ import annotations

import ctypes
import os
import time

import numpy as np

from .engine import Engine, LMX_OK, _raise
from .graph import Matching, PhaseTrace, RoundStats

LMX_OPT_DIST_P = 4
LMX_OPT_DIST_RANK = 5

try:   # the reference's own types when it is importable (graph.py's rationale)
    from locmax.bsp import Partition as _RefPartition
    from locmax.bsp import RoundMessages as _RefRoundMessages
except Exception:
    _RefPartition = _RefRoundMessages = None

#: Bytes per candidate record in the reference's accounting (bsp.py:26).
CANDIDATE_RECORD_BYTES = 32

if _RefPartition is not None:
    Partition, RoundMessages = _RefPartition, _RefRoundMessages
else:
    from dataclasses import dataclass

    @dataclass(frozen=True)
    class RoundMessages:
        """bsp.py:29-41: the reference's per-round boundary accounting."""

        round_index: int
        candidate_records: int
        bytes_estimate: int
        cut_edges_surviving: int
        status_records: int

    @dataclass(frozen=True)
    class Partition:
        """bsp.py:44-57."""

        num_workers: int
        bounds: np.ndarray
        owner: np.ndarray
        local_edges: list
        cut_edges: np.ndarray
        degree_imbalance: float

        @property
        def cut_fraction(self) -> float:
            total = sum(int(e.size) for e in self.local_edges)
            m = total - int(self.cut_edges.size)
            return self.cut_edges.size / m if m else 0.0


def partition_graph(g, p: int):
    """``partition_graph(g, p)`` (bsp.py:60-98): p contiguous vertex ranges
    with near-equal degree sums -- the ranges the B200 partitions own (the
    device computes the same cuts in lmx_setup.cu:partition_bounds)."""
    n = int(g.num_vertices)
    if p < 1:
        raise ValueError("p must be >= 1")
    if p > n:
        raise ValueError(f"p={p} exceeds the vertex count {n}")
    eu = np.asarray(g.edge_u, dtype=np.int64)
    ev = np.asarray(g.edge_v, dtype=np.int64)
    m = int(eu.size)
    deg = np.bincount(eu, minlength=n) + np.bincount(ev, minlength=n)
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(deg, out=offsets[1:])
    two_m = 2 * m
    targets = (np.arange(1, p, dtype=np.float64) * two_m) / p
    cuts = np.searchsorted(offsets, targets, side="left").astype(np.int64)
    if cuts.size:
        steps = np.arange(1, p, dtype=np.int64)
        cuts = np.maximum.accumulate(cuts - steps) + steps
        cuts = np.minimum(np.maximum(cuts, steps), n - p + steps)
        bounds = np.concatenate([[0], cuts, [n]]).astype(np.int64)
    else:
        bounds = np.array([0, n], dtype=np.int64)
    owner = np.repeat(np.arange(p, dtype=np.int64), np.diff(bounds))
    ou, ov = owner[eu], owner[ev]
    ids = np.arange(m, dtype=np.int64)
    local = [ids[(ou == k) | (ov == k)] for k in range(p)]
    cut = ids[ou != ov]
    if two_m:
        share = two_m / p
        imbalance = max(float(offsets[bounds[k + 1]] - offsets[bounds[k]]) for k in range(p)) / share
    else:
        imbalance = 1.0
    return Partition(p, bounds, owner, local, cut, imbalance)


def _bind(lib):
    if getattr(lib, "_dist_bound", False):
        return
    p, i64, u64, c_int = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
    sig = {
        "lmx_dist_bounds": (c_int, [p, p]),
        "lmx_dist_begin": (c_int, [p, u64, c_int]),
        "lmx_dist_round": (c_int, [p]),
        "lmx_dist_propose": (c_int, [p, ctypes.POINTER(p), ctypes.POINTER(p)]),
        "lmx_dist_recv_buffer": (c_int, [p, i64, ctypes.POINTER(p)]),
        "lmx_dist_accept": (c_int, [p, i64]),
        "lmx_dist_match": (c_int, [p, ctypes.POINTER(p)]),
        "lmx_dist_state": (c_int, [p, ctypes.POINTER(p), ctypes.POINTER(p), ctypes.POINTER(p),
                                   ctypes.POINTER(p)]),
        "lmx_dist_mround": (c_int, [p, ctypes.POINTER(p)]),
        "lmx_dist_hist": (c_int, [p, c_int, ctypes.POINTER(p), ctypes.POINTER(c_int)]),
        "lmx_dist_messages": (c_int, [p, c_int, ctypes.POINTER(p)]),
        "lmx_dist_rmat_build": (c_int, [p, c_int, c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double, u64,
                                        c_int, ctypes.POINTER(p), ctypes.POINTER(i64), ctypes.POINTER(p),
                                        ctypes.POINTER(p)]),
        "lmx_dist_rmat_route": (c_int, [p, ctypes.POINTER(p), p, ctypes.POINTER(i64)]),
        "lmx_dist_rmat_recv_buffer": (c_int, [p, i64, ctypes.POINTER(p)]),
        "lmx_dist_rmat_finish": (c_int, [p, c_int]),
        "lmx_dist_load_local": (c_int, [p, i64, i64, p, i64, p, c_int]),
        "lmx_dist_pad": (c_int, [p, i64, ctypes.POINTER(p), ctypes.POINTER(p)]),
        "lmx_dist_list_size": (c_int, [p, ctypes.POINTER(p)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    lib._dist_bound = True


class _CudaBuf:
    """Zero-copy torch view of device memory owned by liblmx."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def _view(ptr: int, shape, typestr: str, device):
    import torch
    if int(np.prod(shape)) == 0:
        dt = {"<i4": torch.int32, "<i8": torch.int64}[typestr]
        return torch.empty(shape, dtype=dt, device=device)
    return torch.as_tensor(_CudaBuf(ptr, shape, typestr), device=device)


class DistRank:
    """One partition: a liblmx context loaded with LMX_OPT_DIST_P / RANK."""

    def __init__(self, g, p: int, rank: int, device: int = 0, stream=None, rmat: dict | None = None,
                 algo: str = "auto", defer: bool = False):
        """Load partition `rank` of `p` from a host graph `g`, or, with
        ``rmat=dict(scale=..., edge_factor=..., seed=...)``, from the device
        RMAT generator (every rank generates the same graph and keeps its part).
        ``algo`` picks the round loop as ``Engine.set_algo`` does ("auto":
        the scan loop when the weights are distinct).  ``defer=True`` only
        creates the context: ``build_rmat_distributed`` then loads it."""
        import torch
        self.eng = Engine(device)
        self.lib = self.eng._lib
        _bind(self.lib)
        self.p, self.rank, self.device = p, rank, torch.device("cuda", device)
        # the device views handed back (counts, records, statistics) are consumed
        # by torch ops / NCCL on torch's current stream: the engine must run on it
        if stream is None:
            stream = torch.cuda.current_stream(self.device).cuda_stream
        self.eng.set_stream(stream)
        self._opt(LMX_OPT_DIST_P, p)
        self._opt(LMX_OPT_DIST_RANK, rank)
        self.eng.set_algo(algo)
        if defer:
            return
        if rmat is not None:
            self.eng.gen_rmat(**rmat)
        else:
            self.eng.load_graph(g)
        self._after_load()

    def _after_load(self):
        p, rank = self.p, self.rank
        self.n, self.m = self.eng.graph_size()
        b = np.zeros(p + 1, dtype=np.int64)
        self._chk(self.lib.lmx_dist_bounds(self.eng._h, b.ctypes.data), "lmx_dist_bounds")
        self.bounds = b
        self.n_local = int(b[rank + 1] - b[rank])
        bm, mate, eb, st = (ctypes.c_void_p() for _ in range(4))
        self._chk(self.lib.lmx_dist_state(self.eng._h, ctypes.byref(bm), ctypes.byref(mate), ctypes.byref(eb),
                                          ctypes.byref(st)), "lmx_dist_state")
        self.words = (self.n + 31) // 32
        self.bitmap = _view(bm.value, (max(self.words, 1),), "<i4", self.device)
        self.mate = _view(mate.value, (max(self.n, 1),), "<i8", self.device)
        self.ebits = _view(eb.value, ((max(self.m, 1) + 31) // 32,), "<i4", self.device)
        # round loop chosen by the load: "scan" (weight-ordered, distinct weights) or "compact"
        self.algo = self.eng.algo()
        self.mround = None   # match round per vertex (device ids): scan loop, or any loop with p > 1
        if self.algo == "scan" or p > 1:
            mr = ctypes.c_void_p()
            self._chk(self.lib.lmx_dist_mround(self.eng._h, ctypes.byref(mr)), "lmx_dist_mround")
            self.mround = _view(mr.value, (max(self.n, 1),), "<i4", self.device)

    def _opt(self, opt, val):
        self._chk(self.lib.lmx_set_option(self.eng._h, opt, val), "lmx_set_option")

    def _chk(self, rc, what):
        if rc != LMX_OK:
            _raise(rc, f"{what}: " + self.lib.lmx_last_error(self.eng._h).decode())

    def begin(self, seed: int, rerandomize: bool):
        self._chk(self.lib.lmx_dist_begin(self.eng._h, seed & ((1 << 64) - 1), int(rerandomize)), "lmx_dist_begin")

    def round(self):
        self._chk(self.lib.lmx_dist_round(self.eng._h), "lmx_dist_round")

    def _cached_view(self, ptr: int, rows: int, cols: int, typestr: str):
        """A tensor over device memory the context owns; the per-round protocol
        asks for the same few buffers every round, so their views are kept
        (a view of at least `rows` rows is sliced)."""
        cache = self.__dict__.setdefault("_view_cache", {})
        key = (ptr, cols, typestr)
        t = cache.get(key)
        if t is None or t.shape[0] < rows:
            t = _view(ptr, (rows, cols) if cols else (rows,), typestr, self.device)
            if rows:
                cache[key] = t
        return t[:rows]

    def propose(self):
        """Exchange-A records on the device: (packed int32 [cap, 2] view, int64[p] counts).
        Nothing is synchronised; the first `counts.sum()` rows are valid."""
        cptr = ctypes.c_void_p()
        sptr = ctypes.c_void_p()
        self._chk(self.lib.lmx_dist_propose(self.eng._h, ctypes.byref(cptr), ctypes.byref(sptr)), "lmx_dist_propose")
        counts = self._cached_view(cptr.value, self.p, 0, "<i8")
        send = self._cached_view(sptr.value, max(self.n_local, 1), 2, "<i4")
        return send, counts

    def pad(self, capacity: int):
        """Fixed-capacity exchange A (lmx_dist_pad, after propose): int32
        [p * capacity, 2] records, destination j's in slot j, and the device
        overflow flag (int32 [1], nonzero if capacity did not bound a count)."""
        pp, op = ctypes.c_void_p(), ctypes.c_void_p()
        self._chk(self.lib.lmx_dist_pad(self.eng._h, int(capacity), ctypes.byref(pp), ctypes.byref(op)),
                  "lmx_dist_pad")
        return (self._cached_view(pp.value, self.p * int(capacity), 2, "<i4"),
                self._cached_view(op.value, 1, 0, "<i4"))

    def list_size(self):
        """This rank's list size for the next round (device int32 [1]; after match)."""
        sp = ctypes.c_void_p()
        self._chk(self.lib.lmx_dist_list_size(self.eng._h, ctypes.byref(sp)), "lmx_dist_list_size")
        return _view(sp.value, (1,), "<i4", self.device)

    def recv_buffer(self, count: int):
        ptr = ctypes.c_void_p()
        self._chk(self.lib.lmx_dist_recv_buffer(self.eng._h, int(count), ctypes.byref(ptr)), "lmx_dist_recv_buffer")
        return self._cached_view(ptr.value, int(count), 2, "<i4")

    def accept(self, count: int):
        self._chk(self.lib.lmx_dist_accept(self.eng._h, int(count)), "lmx_dist_accept")

    def match(self):
        """Enqueue the match step; returns the round's device {live slots, matched} (int64[2] view)."""
        ptr = ctypes.c_void_p()
        self._chk(self.lib.lmx_dist_match(self.eng._h, ctypes.byref(ptr)), "lmx_dist_match")
        return self._cached_view(ptr.value, 2, 0, "<i8")

    def word_range(self, k: int):
        return int(self.bounds[k]) // 32, (int(self.bounds[k + 1]) + 31) // 32

    def vertex_range(self, k: int):
        return int(self.bounds[k]), int(self.bounds[k + 1])

    def hist(self, n_rounds: int):
        """Scan loop: this partition's death-round histogram (device int64 view)."""
        hp = ctypes.c_void_p()
        nb = ctypes.c_int()
        self._chk(self.lib.lmx_dist_hist(self.eng._h, int(n_rounds), ctypes.byref(hp), ctypes.byref(nb)),
                  "lmx_dist_hist")
        return _view(hp.value, (nb.value,), "<i8", self.device)

    def messages(self, n_rounds: int):
        """This partition's share of the reference's boundary accounting
        (lmx_dist_messages): device uint64 [2, n_rounds + 1] = candidate records
        by last round sent, cut edges by death round.  Needs the all-gathered
        match rounds."""
        hp = ctypes.c_void_p()
        self._chk(self.lib.lmx_dist_messages(self.eng._h, int(n_rounds), ctypes.byref(hp)), "lmx_dist_messages")
        return _view(hp.value, (2 * (n_rounds + 1),), "<i8", self.device)

    def load_local_edges(self, records, count: int, degrees, m: int):
        """Load this partition from host memory (lmx_dist_load_local):
        `records` (int32 [>= count, 6], page-locked) are its local edges with
        their global ids, `degrees` (int32 [n], page-locked) the global degrees
        in caller ids, `m` the global edge count -- as
        ``build_rmat_distributed(..., keep_records=True)`` keeps them.  The
        host-to-device copies and the partition's K0 run on the engine's stream."""
        self._chk(self.lib.lmx_dist_load_local(self.eng._h, int(degrees.numel()), int(m), degrees.data_ptr(),
                                               int(count), records.data_ptr() if count else None, self.w_uniform),
                  "lmx_dist_load_local")
        self._after_load()

    def close(self):
        self.eng.close()


def build_rmat_distributed(ranks, comm, scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19,
                           c: float = 0.19, seed: int = 1, permute: bool = True, keep_records: bool = False):
    """Load the local partitions ``ranks`` (created with ``defer=True``) with the
    RMAT graph of ``lmx_gen_rmat``'s recipe WITHOUT any rank holding the whole
    graph (config C5): each rank builds the pairs that hash to it (an even
    share whatever the ids), the first-occurrence bitmaps and the degrees are summed over
    the ranks (the global edge ids and partition_graph's cuts follow), and
    every pair is sent to the owners of its ends (all-to-all-v).
    ``keep_records=True`` also keeps each rank's received records -- its
    local edges (bsp.py:86-90) with their global ids -- in page-locked host
    memory (``rank.host_records``), so ``DistRank.load_local_edges`` can load
    the partition again from the host (the multi-GPU end-to-end leg)."""
    import torch
    bits, degs, mms = [], [], []
    for r in ranks:
        bp, dp, mp = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        words = ctypes.c_int64()
        r._chk(r.lib.lmx_dist_rmat_build(r.eng._h, scale, edge_factor, a, b, c, seed & ((1 << 64) - 1),
                                         int(permute), ctypes.byref(bp), ctypes.byref(words), ctypes.byref(dp),
                                         ctypes.byref(mp)), "lmx_dist_rmat_build")
        bits.append(_view(bp.value, (max(words.value, 1),), "<i4", r.device))
        degs.append(_view(dp.value, (1 << scale,), "<i4", r.device))
        mms.append(_view(mp.value, (2,), "<i8", r.device))
    # disjoint bit sets: an int32 sum is their OR; degree contributions add
    comm.allreduce_sum_(ranks, bits)
    comm.allreduce_sum_(ranks, degs)
    if keep_records:   # the global degrees (caller ids): partition_graph's cuts on a reload
        for r, d in zip(ranks, degs):
            r.host_degrees = torch.empty(d.shape, dtype=torch.int32, pin_memory=True)
            r.host_degrees.copy_(d)
    lo = comm.allreduce_min_u64(ranks, [m_[0:1] for m_ in mms])
    hi = comm.allreduce_max_u64(ranks, [m_[1:2] for m_ in mms])
    uniform = int(lo == hi)
    sends = []
    for r in ranks:
        sp = ctypes.c_void_p()
        counts = np.zeros(r.p, dtype=np.int64)
        mtot = ctypes.c_int64()
        r._chk(r.lib.lmx_dist_rmat_route(r.eng._h, ctypes.byref(sp), counts.ctypes.data, ctypes.byref(mtot)),
               "lmx_dist_rmat_route")
        total = int(counts.sum())
        sends.append((_view(sp.value, (max(total, 1), 6), "<i4", r.device), counts))
    recvs = comm.alltoallv_records(ranks, sends, 6, lambda r, cnt: _recv_records(r, cnt))
    for r, cnt in zip(ranks, recvs):
        r.w_uniform = uniform
        if keep_records:
            h = torch.empty((max(int(cnt), 1), 6), dtype=torch.int32, pin_memory=True)
            if cnt:
                h[:cnt].copy_(_recv_records(r, cnt, keep=True)[:cnt])
            r.host_records = (h, int(cnt))
        r._chk(r.lib.lmx_dist_rmat_finish(r.eng._h, uniform), "lmx_dist_rmat_finish")
        r._after_load()
    torch.cuda.synchronize()


def _recv_records(r, count: int, keep: bool = False):
    """The device buffer of `count` received build records (allocated by
    liblmx; ``keep=True``: the one already allocated, records intact)."""
    if keep:
        return _view(r._recv_ptr, (max(int(count), 1), 6), "<i4", r.device)
    rp = ctypes.c_void_p()
    r._chk(r.lib.lmx_dist_rmat_recv_buffer(r.eng._h, int(count), ctypes.byref(rp)), "lmx_dist_rmat_recv_buffer")
    r._recv_ptr = rp.value
    return _view(rp.value, (max(int(count), 1), 6), "<i4", r.device)


class LocalComm:
    """All p partitions in this process (one GPU): collectives are device copies."""

    def __init__(self, p: int):
        self.p = p

    def record_total(self, recv_counts):
        return int(sum(recv_counts))

    def alltoallv(self, ranks, sends):
        import torch
        counts_h = [c.tolist() for _, c in sends]
        recvs = []
        for dst in range(self.p):
            parts = []
            for src in range(self.p):
                send, _ = sends[src]
                counts = counts_h[src]
                off = int(sum(counts[:dst]))
                parts.append(send[off: off + int(counts[dst])])
            total = sum(int(x.shape[0]) for x in parts)
            buf = ranks[dst].recv_buffer(total)
            if total:
                buf.copy_(torch.cat(parts, dim=0))
            recvs.append(total)
        return recvs

    def allgather_bitmap(self, ranks):
        # ranges follow bsp.py's cuts, so a boundary word holds bits of two
        # ranks: merge by OR (a bit is only ever set, by its owner)
        for src in range(self.p):
            w0, w1 = ranks[src].word_range(src)
            if w1 <= w0:
                continue
            seg = ranks[src].bitmap[w0:w1]
            for dst in range(self.p):
                if dst != src:
                    ranks[dst].bitmap[w0:w1].bitwise_or_(seg)

    def allgather_mround(self, ranks):
        for src in range(self.p):
            a, b = ranks[src].vertex_range(src)
            if b <= a:
                continue
            seg = ranks[src].mround[a:b]
            for dst in range(self.p):
                if dst != src:
                    ranks[dst].mround[a:b].copy_(seg)

    def allreduce_sum(self, values):
        return [sum(col) for col in zip(*(v.tolist() for v in values))]

    def allreduce_sum_(self, ranks, tensors):
        total = tensors[0].clone()
        for t in tensors[1:]:
            total += t
        for t in tensors:
            t.copy_(total)

    def allreduce_min_u64(self, ranks, tensors):
        return min(int(t.item()) & ((1 << 64) - 1) for t in tensors)

    def allreduce_max_u64(self, ranks, tensors):
        return max(int(t.item()) & ((1 << 64) - 1) for t in tensors)

    def alltoallv_records(self, ranks, sends, width, recv_buffer):
        """sends[k] = (records [*, width] int32 packed by destination, int64 counts[p])."""
        import torch
        counts_h = [c.tolist() if hasattr(c, "tolist") else list(c) for _, c in sends]
        out = []
        for dst in range(self.p):
            parts = []
            for src in range(self.p):
                off = int(sum(counts_h[src][:dst]))
                parts.append(sends[src][0][off: off + int(counts_h[src][dst])])
            total = sum(int(x.shape[0]) for x in parts)
            buf = recv_buffer(ranks[dst], total)
            if total:
                buf[:total].copy_(torch.cat(parts, dim=0))
            out.append(total)
        return out

    def gather_outputs(self, ranks):
        import torch
        mate = ranks[0].mate.clone()
        ebits = ranks[0].ebits.clone()
        for r in ranks[1:]:
            mate = torch.maximum(mate, r.mate)
            ebits = ebits | r.ebits
        return mate, ebits


class TorchComm:
    """One partition per process under torch.distributed (nccl or gloo)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.p = dist.get_world_size()
        self.rank = dist.get_rank()

    def alltoallv(self, ranks, sends):
        import torch
        (me,), ((send, counts),) = ranks, sends
        dev = me.device
        sc = torch.as_tensor(counts, dtype=torch.int64, device=dev)
        rc = torch.empty_like(sc)
        self.dist.all_to_all_single(rc, sc)
        both = torch.cat([sc, rc]).tolist()          # the one host sync of exchange A
        scounts, rcounts = both[: self.p], both[self.p:]
        stotal, total = int(sum(scounts)), int(sum(rcounts))
        recv = me.recv_buffer(total)
        flat_in = send[:stotal].reshape(-1) if stotal else torch.empty(0, dtype=torch.int32, device=dev)
        flat_out = recv.reshape(-1) if total else torch.empty(0, dtype=torch.int32, device=dev)
        self.dist.all_to_all_single(flat_out, flat_in, [2 * c for c in rcounts], [2 * int(c) for c in scounts])
        return [total]

    def alltoallv_stats(self, ranks, sends, prev):
        """Exchange A of round r with round r-1's statistics riding along.

        `prev` is round r-1's device {candidates found, matched vertices}
        (None in round 0).  Every rank sends its own pair to every peer next
        to the record count, so one all-to-all and ONE host read give both
        this round's record counts and the global statistics of the last
        round (the separate all-reduce and its host sync are gone).  Returns
        ([records received], (found, matched) of round r-1 or None); when the
        last round found no candidate anywhere, the records are not exchanged
        (every count is zero then: each list is empty).
        """
        import torch
        (me,), ((send, counts),) = ranks, sends
        dev = me.device
        bufs = getattr(self, "_stats_bufs", None)
        if bufs is None or bufs[0].device != dev:
            sc = torch.zeros((self.p, 3), dtype=torch.int64, device=dev)
            both_d = torch.empty(4 * self.p, dtype=torch.int64, device=dev)   # [send counts | received rows]
            both_h = torch.empty(4 * self.p, dtype=torch.int64, pin_memory=torch.device(dev).type == "cuda")
            self._stats_bufs = bufs = (sc, both_d, both_h)
        sc, both_d, both_h = bufs
        sc[:, 0].copy_(counts)
        if prev is not None:
            sc[:, 1:].copy_(prev.reshape(1, 2).expand(self.p, 2))
        else:
            sc[:, 1:].zero_()
        both_d[: self.p].copy_(counts)
        self.dist.all_to_all_single(both_d[self.p:], sc.reshape(-1))
        both_h.copy_(both_d)
        both = both_h.tolist()   # (the copy above is synchronous: the one host sync of the round)
        scounts = both[: self.p]
        rows = [both[self.p + 3 * k: self.p + 3 * k + 3] for k in range(self.p)]
        rcounts = [r[0] for r in rows]
        stats = None if prev is None else (int(sum(r[1] for r in rows)), int(sum(r[2] for r in rows)))
        if stats is not None and stats[0] == 0:
            return [0], stats
        stotal, total = int(sum(scounts)), int(sum(rcounts))
        recv = me.recv_buffer(total)
        flat_in = send[:stotal].reshape(-1) if stotal else torch.empty(0, dtype=torch.int32, device=dev)
        flat_out = recv.reshape(-1) if total else torch.empty(0, dtype=torch.int32, device=dev)
        self.dist.all_to_all_single(flat_out, flat_in, [2 * c for c in rcounts], [2 * int(c) for c in scounts])
        return [total], stats

    def allgather_bitmap(self, ranks):
        import torch
        (me,) = ranks
        # exchange B runs every round: the spans and the padded send/receive
        # buffers are kept per partition (the pad words stay zero)
        spans = tuple(me.word_range(k) for k in range(self.p))
        key = (spans, str(me.bitmap.device))
        cache = getattr(self, "_bm_cache", None)
        if cache is None or cache[0] != key:
            width = max(max(w1 - w0 for w0, w1 in spans), 1)
            row = torch.zeros(width, dtype=torch.int32, device=me.device)
            out = torch.empty(self.p * width, dtype=torch.int32, device=me.device)
            self._bm_cache = cache = (key, row, out, spans, width)
        _, row, out, spans, width = cache
        w0, w1 = spans[self.rank]
        if w1 > w0:
            row[: w1 - w0].copy_(me.bitmap[w0:w1])
        self.dist.all_gather_into_tensor(out, row)
        for k, (a, b) in enumerate(spans):
            if k != self.rank and b > a:   # boundary words are shared: OR
                me.bitmap[a:b].bitwise_or_(out[k * width: k * width + (b - a)])

    def allgather_mround(self, ranks):
        import torch
        (me,) = ranks
        spans = [me.vertex_range(k) for k in range(self.p)]
        width = max(max(b - a for a, b in spans), 1)
        a, b = spans[self.rank]
        row = torch.zeros(width, dtype=torch.int32, device=me.device)
        if b > a:
            row[: b - a].copy_(me.mround[a:b])
        out = torch.empty(self.p * width, dtype=torch.int32, device=me.device)
        self.dist.all_gather_into_tensor(out, row)
        for k, (x, y) in enumerate(spans):
            if k != self.rank and y > x:
                me.mround[x:y].copy_(out[k * width: k * width + (y - x)])

    def allreduce_sum(self, values):
        (vals,) = values
        t = vals.clone()   # device int64[k]
        self.dist.all_reduce(t)
        return [int(x) for x in t.tolist()]

    def allreduce_sum_(self, ranks, tensors):
        (t,) = tensors
        self.dist.all_reduce(t)

    def allreduce_max_(self, ranks, tensors):
        (t,) = tensors
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)

    def _u64_extreme(self, tensors, op):
        import torch
        (t,) = tensors
        # u64 weight bits of non-negative doubles stay below 2^63: int64 compare is exact
        x = t.clone()
        self.dist.all_reduce(x, op=op)
        return int(x.item()) & ((1 << 64) - 1)

    def allreduce_min_u64(self, ranks, tensors):
        return self._u64_extreme(tensors, self.dist.ReduceOp.MIN)

    def allreduce_max_u64(self, ranks, tensors):
        return self._u64_extreme(tensors, self.dist.ReduceOp.MAX)

    def alltoallv_records(self, ranks, sends, width, recv_buffer):
        import torch
        (me,), ((send, counts),) = ranks, sends
        dev = me.device
        sc = torch.as_tensor(np.asarray(counts), dtype=torch.int64, device=dev)
        rc = torch.empty_like(sc)
        self.dist.all_to_all_single(rc, sc)
        scounts, rcounts = [int(x) for x in sc.tolist()], [int(x) for x in rc.tolist()]
        total = sum(rcounts)
        recv = recv_buffer(me, total)
        flat_in = send[: sum(scounts)].reshape(-1)
        flat_out = recv[:total].reshape(-1) if total else torch.empty(0, dtype=torch.int32, device=dev)
        self.dist.all_to_all_single(flat_out, flat_in, [width * c for c in rcounts], [width * c for c in scounts])
        return [total]

    def alltoall_padded(self, ranks, padded, counts, capacity: int):
        """Exchange A with equal, host-known splits (p slots of `capacity`
        records; filler skipped by accept): no host round trip.  Returns the
        slots' record total (what accept reads) and this rank's received
        record count as a device int64 [1]."""
        import torch
        (me,) = ranks
        total = self.p * int(capacity)
        recv = me.recv_buffer(total)
        self.dist.all_to_all_single(recv.reshape(-1), padded[:total].reshape(-1))
        rc = torch.empty_like(counts)
        self.dist.all_to_all_single(rc, counts)
        return total, rc.sum().view(1)

    def gather_outputs(self, ranks):
        """The global mate table and matched-edge bits on every rank.  Each
        rank writes mate only inside its owned range (relabelling stays inside
        a range), so the owned slices are all-gathered: (p-1)/p of n int64 per
        rank instead of an all-reduce's 2 (p-1)/p.  The edge bits are set by
        the owner of an edge's lower end, scattered over the id space: an
        all-reduce (disjoint bit sets: sum == or)."""
        import torch
        (me,) = ranks
        spans = [me.vertex_range(k) for k in range(self.p)]
        width = max(max(b - a for a, b in spans), 1)
        a, b = spans[self.rank]
        row = torch.full((width,), -1, dtype=torch.int64, device=me.device)
        if b > a:
            row[: b - a].copy_(me.mate[a:b])
        out = torch.empty(self.p * width, dtype=torch.int64, device=me.device)
        self.dist.all_gather_into_tensor(out, row)
        mate = torch.full_like(me.mate, -1)
        for k, (x, y) in enumerate(spans):
            if y > x:
                mate[x:y].copy_(out[k * width: k * width + (y - x)])
        ebits = me.ebits.clone()
        self.dist.all_reduce(ebits)
        return mate, ebits

    def bind_device(self, device):
        self._dev = device

    def record_total(self, recv_counts):
        """Exchange-A records received by this rank (the per-rank share of RoundMessages)."""
        return int(sum(recv_counts))


def run_rounds(ranks, comm, seed: int, rerandomize: bool = True, max_rounds: int | None = None):
    """Drive the stepped protocol on `ranks` (all local partitions) to completion.

    Returns (RoundStats list, per-round exchange-A record counts).  Host
    synchronisations per round: the exchange-A counts and the statistics
    all-reduce (termination).
    """
    algos = {r.algo for r in ranks}
    if len(algos) != 1:
        raise RuntimeError(f"internal: partitions disagree on the round loop {sorted(algos)}")
    if algos == {"scan"}:
        return _run_rounds_scan(ranks, comm, seed, rerandomize, max_rounds)
    for r in ranks:
        r.begin(seed, rerandomize)
    before = []
    matched = []
    records = []
    while True:
        for r in ranks:
            r.round()
        sends = [r.propose() for r in ranks]
        recv_counts = comm.alltoallv(ranks, sends)
        records.append(comm.record_total(recv_counts))
        for r, cnt in zip(ranks, recv_counts):
            r.accept(cnt)
        local = [r.match() for r in ranks]
        comm.allgather_bitmap(ranks)
        live, mv = comm.allreduce_sum(local)
        if live == 0:
            records.pop()
            break
        if live % 2 or mv % 2:
            raise RuntimeError("internal: odd global slot or matched-vertex count")
        before.append(live // 2)
        matched.append(mv // 2)
        if max_rounds is not None and len(before) > max_rounds:
            raise RuntimeError("round limit exceeded")
    stats = []
    for i, b in enumerate(before):
        nxt = before[i + 1] if i + 1 < len(before) else 0
        stats.append(RoundStats(b, matched[i], b - nxt))
    if ranks[0].mround is not None:   # every partition's match rounds, for round_messages()
        comm.allgather_mround(ranks)
    return stats, records


def round_messages(ranks, comm, n_rounds: int) -> list:
    """``trace.messages`` of bsp_local_max (bsp.py:148-199): per round the
    candidate records (deduplicated per (vertex, receiving worker)), their
    32-byte estimate, the surviving cut edges and the 2-per-cut-edge status
    records -- derived on the device from the edges' death rounds
    (lmx_dist_messages) and summed over the partitions."""
    p = ranks[0].p
    if p == 1 or n_rounds == 0:
        return [RoundMessages(r, 0, 0, 0, 0) for r in range(n_rounds)]
    h = comm.allreduce_sum([r.messages(n_rounds) for r in ranks])
    rec, cut = h[: n_rounds + 1], h[n_rounds + 1:]
    out = []
    rs = cs = 0
    suff_rec = [0] * (n_rounds + 1)
    suff_cut = [0] * (n_rounds + 1)
    for d in range(n_rounds, -1, -1):
        rs += rec[d]
        cs += cut[d]
        suff_rec[d], suff_cut[d] = rs, cs
    for r in range(n_rounds):
        out.append(RoundMessages(r, suff_rec[r], suff_rec[r] * CANDIDATE_RECORD_BYTES, suff_cut[r],
                                 2 * suff_cut[r]))
    return out


def _run_rounds_scan(ranks, comm, seed: int, rerandomize: bool, max_rounds: int | None):
    """The protocol on the weight-ordered scan loop (lmx_scan.cu): the loop ends
    when no partition finds a candidate; RoundStats come afterwards from the
    summed death-round histograms (each edge counted by the owner of its
    higher end), as in the single-GPU scan loop."""
    for r in ranks:
        r.begin(seed, rerandomize)
    matched = []
    records = []
    if hasattr(comm, "alltoallv_stats"):
        # One host sync per round: round r's exchange A carries round r-1's
        # statistics.  The round after the last one (no candidate anywhere)
        # is probed and proposed on empty lists -- A_{r+1} holds only
        # vertices that found a candidate -- and stops before its match step.
        prev = None
        while True:
            for r in ranks:
                r.round()
            sends = [r.propose() for r in ranks]
            recv_counts, st = comm.alltoallv_stats(ranks, sends, prev)
            if st is not None:
                found, mv = st
                if found == 0:
                    records.pop()
                    break
                if mv % 2:
                    raise RuntimeError("internal: odd global matched-vertex count")
                matched.append(mv // 2)
                if max_rounds is not None and len(matched) > max_rounds:
                    raise RuntimeError("round limit exceeded")
            records.append(comm.record_total(recv_counts))
            for r, cnt in zip(ranks, recv_counts):
                r.accept(cnt)
            (prev,) = [r.match().clone() for r in ranks]   # the view lives in the counter array
            comm.allgather_bitmap(ranks)
            if (st is not None and st[0] <= _LATE_FOUND and hasattr(comm, "alltoall_padded")
                    and all(r.algo == "scan" and hasattr(r, "pad") for r in ranks)):
                _late_rounds(ranks, comm, prev, matched, records, max_rounds)
                break
    else:
        while True:
            for r in ranks:
                r.round()
            sends = [r.propose() for r in ranks]
            recv_counts = comm.alltoallv(ranks, sends)
            records.append(comm.record_total(recv_counts))
            for r, cnt in zip(ranks, recv_counts):
                r.accept(cnt)
            local = [r.match() for r in ranks]
            comm.allgather_bitmap(ranks)
            found, mv = comm.allreduce_sum(local)
            if found == 0:
                records.pop()
                break
            if mv % 2:
                raise RuntimeError("internal: odd global matched-vertex count")
            matched.append(mv // 2)
            if max_rounds is not None and len(matched) > max_rounds:
                raise RuntimeError("round limit exceeded")
    n_rounds = len(matched)
    comm.allgather_mround(ranks)
    hist = comm.allreduce_sum([r.hist(n_rounds) for r in ranks])
    m = ranks[0].m
    if hist[n_rounds] != 0 or sum(hist) != m:
        raise RuntimeError(f"internal: death-round histogram covers {sum(hist)} of {m} edges, "
                           f"{hist[n_rounds]} outlived the loop")
    stats = []
    alive = m
    for i in range(n_rounds):
        stats.append(RoundStats(alive, matched[i], hist[i]))
        alive -= hist[i]
    return stats, records


#: The late rounds (global candidates found in a round at most this many)
#: run in batches of _LATE_BATCH with fixed-capacity exchanges and one host
#: round trip per batch instead of one per round.
_LATE_FOUND = int(os.environ.get("LMX_DIST_LATE_FOUND", str(1 << 22)))
_LATE_BATCH = max(1, int(os.environ.get("LMX_DIST_LATE_BATCH", "8")))


def _late_rounds(ranks, comm, prev, matched, records, max_rounds):
    """The tail of the round protocol (scan loop partitions, TorchComm).

    The lists only shrink, so the largest list of any rank now bounds every
    rank's exchange-A count in every later round: exchange A runs with that
    fixed capacity per destination (lmx_dist_pad; equal all-to-all splits the
    host knows), and a batch of rounds is enqueued with no host round trip.
    Their statistics come back in one all-reduce per batch; rounds enqueued
    past the end (no candidate anywhere) probe and match empty lists.
    `prev` is the last synchronised round's pending {found, matched} (device)."""
    import torch
    (me,) = ranks
    cap = me.list_size().to(torch.int64)
    comm.allreduce_max_(ranks, [cap])
    capacity = max(int(cap.item()), 1)
    rows, recs = [prev], []   # per round: {found, matched} (summed over ranks) / records received here
    first = True
    while True:
        for _ in range(_LATE_BATCH):
            me.round()
            _send, counts = me.propose()
            padded, overflow = me.pad(capacity)
            total, received = comm.alltoall_padded(ranks, padded, counts, capacity)
            me.accept(total)
            rows.append(me.match().clone())
            recs.append(received)
            comm.allgather_bitmap(ranks)
        flat = torch.cat([torch.stack(rows).reshape(-1), overflow.to(torch.int64)])
        comm.allreduce_sum_(ranks, [flat])
        h = torch.cat([flat] + recs).tolist()   # the batch's one host round trip
        nrow = len(rows)
        if h[2 * nrow]:
            raise RuntimeError("internal: exchange-A capacity exceeded")
        rec_h = h[2 * nrow + 1:]
        skip = 1 if first else 0   # the first batch starts with the synchronised round (its records are in)
        for i in range(nrow):
            found, mv = h[2 * i], h[2 * i + 1]
            if found == 0:
                if i < skip:
                    records.pop()
                return
            if mv % 2:
                raise RuntimeError("internal: odd global matched-vertex count")
            matched.append(mv // 2)
            if i >= skip:
                records.append(int(rec_h[i - skip]))
            if max_rounds is not None and len(matched) > max_rounds:
                raise RuntimeError("round limit exceeded")
        rows, recs = [], []
        first = False


def _unpack_ids(ebits, m: int) -> np.ndarray:
    words = ebits.cpu().numpy().view(np.uint32)
    bits = np.unpackbits(words.view(np.uint8), bitorder="little")[:m]
    return np.nonzero(bits)[0].astype(np.int64)


def local_max_dist(g, p: int, seed: int, rerandomize: bool = True, device: int = 0, algo: str = "auto"):
    """Drop-in for ``bsp_local_max(g, p, seed, rerandomize)`` (bsp.py:101-205):
    p partitions emulated in this process on one B200.  ``trace.messages``
    holds the reference's ``RoundMessages`` per round (bsp.py:29-41,
    :148-199), identical to bsp_local_max's; ``trace.exchange_a_records`` the
    records this engine actually exchanged."""
    import torch
    t0 = time.perf_counter()
    if p < 1:
        raise ValueError("p must be >= 1")
    if p > max(g.num_vertices, 1):
        raise ValueError(f"p={p} exceeds the vertex count {g.num_vertices}")
    torch.cuda.set_device(device)
    stream = torch.cuda.current_stream(device).cuda_stream
    ranks = [DistRank(g, p, k, device, stream, algo=algo) for k in range(p)]
    try:
        comm = LocalComm(p)
        stats, records = run_rounds(ranks, comm, seed, rerandomize)
        messages = round_messages(ranks, comm, len(stats))
        mate, ebits = comm.gather_outputs(ranks)
        ids = _unpack_ids(ebits, ranks[0].m)
        mate_h = mate.cpu().numpy()[: g.num_vertices].copy()
    finally:
        for r in ranks:
            r.close()
    trace = PhaseTrace(rounds=stats, messages=messages)
    trace.exchange_a_records = records   # this engine's own per-round record counts
    trace.wall_millis = (time.perf_counter() - t0) * 1000.0
    return Matching(ids, mate_h), trace


def local_max_dist_rmat(p: int, scale: int, seed: int, rerandomize: bool = True, edge_factor: int = 16,
                        a: float = 0.57, b: float = 0.19, c: float = 0.19, graph_seed: int = 1,
                        permute: bool = True, device: int = 0):
    """p partitions in this process, built by the distributed RMAT builder
    (no rank ever holds the whole graph), then the bsp_local_max protocol.
    Returns (Matching, PhaseTrace, per-rank (device bytes after the load,
    high-water mark during it))."""
    import torch
    torch.cuda.set_device(device)
    stream = torch.cuda.current_stream(device).cuda_stream
    ranks = [DistRank(None, p, k, device, stream, defer=True) for k in range(p)]
    try:
        comm = LocalComm(p)
        build_rmat_distributed(ranks, comm, scale, edge_factor, a, b, c, graph_seed, permute)
        dev_bytes = [(r.eng.device_bytes(), r.eng.peak_device_bytes()) for r in ranks]
        stats, records = run_rounds(ranks, comm, seed, rerandomize)
        messages = round_messages(ranks, comm, len(stats))
        mate, ebits = comm.gather_outputs(ranks)
        ids = _unpack_ids(ebits, ranks[0].m)
        mate_h = mate.cpu().numpy()[: ranks[0].n].copy()
    finally:
        for r in ranks:
            r.close()
    trace = PhaseTrace(rounds=stats, messages=messages)
    trace.exchange_a_records = records
    return Matching(ids, mate_h), trace, dev_bytes


def local_max_torchdist(g, seed: int, rerandomize: bool = True):
    """One partition per torch.distributed rank (launch with torchrun, NCCL)."""
    import torch
    import torch.distributed as dist
    comm = TorchComm()
    dev = torch.cuda.current_device()
    comm.bind_device(torch.device("cuda", dev))
    me = DistRank(g, comm.p, comm.rank, dev, torch.cuda.current_stream().cuda_stream)
    try:
        stats, records = run_rounds([me], comm, seed, rerandomize)
        messages = round_messages([me], comm, len(stats))
        mate, ebits = comm.gather_outputs([me])
        ids = _unpack_ids(ebits, me.m) if comm.rank == 0 else None
        mate_h = mate.cpu().numpy()[: g.num_vertices].copy() if comm.rank == 0 else None
    finally:
        me.close()
    dist.barrier()
    trace = PhaseTrace(rounds=stats, messages=messages)
    trace.exchange_a_records = records
    return (Matching(ids, mate_h) if comm.rank == 0 else None), trace
