"""ctypes front end of liblmx.so (include/lmx.h) and the drop-in entry points.

``local_max_b200(g, seed, rerandomize=True)`` has the signature and result
contract of ``locmax.matchers.local_max_seq`` (matchers.py:61-122): same
``Matching`` (edge set + mate table) and the same ``RoundStats`` trace, bit
for bit, computed by the sm_100a kernels in ``csrc/``.  There is no CPU
fallback: if the shared library or a B200 is missing, the call raises.

``run_matcher`` mirrors ``locmax.bench.run_matcher`` (bench.py:119-142) with
the extra engine ``"b200"``.
"""

from __future__ import annotations

import ctypes
import os
import threading
import time

import numpy as np

from .graph import Graph, Matching, MatchingCheck, PhaseTrace, RoundStats

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LMX_LIBRARY") or os.path.join(_HERE, "liblmx.so")
_UINT64_MASK = (1 << 64) - 1

LMX_OK, LMX_EINVAL, LMX_ECUDA, LMX_ENOMEM, LMX_ELIMIT, LMX_ESTATE = range(6)
LMX_HOST, LMX_DEVICE = 0, 1

EXPORTED_SYMBOLS = (
    "lmx_abi_version", "lmx_create", "lmx_destroy", "lmx_last_error", "lmx_set_stream",
    "lmx_load_graph", "lmx_match", "lmx_last_timing", "lmx_last_rounds", "lmx_last_kernel_times", "lmx_last_round_counters",
    "lmx_local_max",
    "lmx_build_graph", "lmx_gen_rmat", "lmx_gen_rmat_raw", "lmx_gen_er", "lmx_gen_rgg", "lmx_graph_size",
    "lmx_graph_export", "lmx_device_bytes", "lmx_set_option", "lmx_validate", "lmx_rbm",
    "lmx_dist_bounds", "lmx_dist_begin", "lmx_dist_round", "lmx_dist_propose", "lmx_dist_recv_buffer",
    "lmx_dist_accept", "lmx_dist_match", "lmx_dist_state", "lmx_dist_mround", "lmx_dist_hist",
    "lmx_dist_messages", "lmx_pram_cross", "lmx_dist_rmat_build", "lmx_dist_rmat_route",
    "lmx_dist_rmat_recv_buffer", "lmx_dist_rmat_finish", "lmx_dist_load_local", "lmx_dist_pad", "lmx_dist_list_size",
    "lmx_mesh_edges", "lmx_ratings", "lmx_contract",
)
LMX_OPT_KERNEL_TIMING = 1
LMX_OPT_LAYOUT = 2
LMX_OPT_RELABEL = 3
LMX_OPT_ALGO = 6
LMX_OPT_STATIC_ORDER = 7
LMX_OPT_STATIC_SEED = 8
LMX_QUERY_STATIC = 104
LMX_QUERY_LAYOUT = 100
LMX_QUERY_RELABELED = 101
LMX_QUERY_ALGO = 102
_CUDA_STREAM_LEGACY = 1   # cudaStreamLegacy


class LmxRoundStats(ctypes.Structure):
    _fields_ = [("edges_before", ctypes.c_int64), ("edges_matched", ctypes.c_int64),
                ("edges_removed", ctypes.c_int64)]


class LmxTiming(ctypes.Structure):
    _fields_ = [("setup_ms", ctypes.c_double), ("rounds_ms", ctypes.c_double),
                ("output_ms", ctypes.c_double), ("round_launches", ctypes.c_int64),
                ("slot_reads", ctypes.c_int64), ("round_kernel_ms", ctypes.c_double),
                ("match_kernel_ms", ctypes.c_double), ("rounds_executed", ctypes.c_int64),
                ("hist_kernel_ms", ctypes.c_double)]


_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load liblmx.so; raises RuntimeError (never falls back) if absent."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"liblmx.so not found at {path}; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (or `make -C paper_1302_4587_b200/csrc`)")
        lib = ctypes.CDLL(path)
        p, i64, u64, c_int = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
        sig = {
            "lmx_abi_version": (c_int, []),
            "lmx_create": (c_int, [c_int, ctypes.POINTER(p)]),
            "lmx_destroy": (None, [p]),
            "lmx_last_error": (ctypes.c_char_p, [p]),
            "lmx_set_stream": (c_int, [p, p]),
            "lmx_load_graph": (c_int, [p, i64, i64, p, p, p, c_int]),
            "lmx_match": (c_int, [p, u64, c_int, p, p, p, p, c_int, p, c_int]),
            "lmx_last_timing": (c_int, [p, ctypes.POINTER(LmxTiming)]),
            "lmx_last_rounds": (c_int, [p, p, c_int]),
            "lmx_last_kernel_times": (c_int, [p, p, c_int]),
            "lmx_last_round_counters": (c_int, [p, p, c_int]),
            "lmx_local_max": (c_int, [c_int, i64, i64, p, p, p, u64, c_int, p, p, p, p, c_int, p,
                                      ctypes.c_char_p, ctypes.c_size_t]),
            "lmx_build_graph": (c_int, [p, i64, p, p, p, i64, c_int]),
            "lmx_gen_rmat": (c_int, [p, c_int, c_int, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, u64, c_int]),
            "lmx_gen_rmat_raw": (c_int, [p, c_int, c_int, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_double, u64, c_int, p, p, p, c_int]),
            "lmx_gen_er": (c_int, [p, c_int, c_int, u64, c_int]),
            "lmx_gen_rgg": (c_int, [p, c_int, u64, u64, u64, u64, ctypes.c_double, c_int]),
            "lmx_graph_size": (c_int, [p, p, p]),
            "lmx_graph_export": (c_int, [p, p, p, p, c_int]),
            "lmx_device_bytes": (i64, [p]),
            "lmx_set_option": (c_int, [p, c_int, i64]),
            "lmx_validate": (c_int, [p, p, p, i64, c_int, p, p, p, p, ctypes.c_size_t]),
            "lmx_rbm": (c_int, [p, u64, p, p, p, p, c_int, p, c_int]),
            "lmx_pram_cross": (c_int, [p, p, p, c_int]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.lmx_abi_version() != 1:
            raise RuntimeError("liblmx.so ABI version mismatch")
        _lib = lib
        return lib


def _raise(code: int, msg: str):
    if code == LMX_EINVAL:
        raise ValueError(msg)
    if code == LMX_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def _ptr(a) -> int:
    """Address of a numpy array or a torch tensor (CUDA or CPU)."""
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


class Engine:
    """One liblmx context bound to a CUDA device (a B200)."""

    def __init__(self, device: int = 0):
        self._lib = load_library()
        h = ctypes.c_void_p()
        rc = self._lib.lmx_create(device, ctypes.byref(h))
        if rc != LMX_OK:
            _raise(rc, "lmx_create failed: " + self._lib.lmx_last_error(None).decode())
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            self._lib.lmx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, rc: int, what: str):
        if rc != LMX_OK:
            _raise(rc, f"{what}: " + self._lib.lmx_last_error(self._h).decode())

    def set_stream(self, stream_handle: int | None):
        """Run on a given cudaStream_t (e.g. ``torch.cuda.current_stream().cuda_stream``).

        ``None`` = the engine's own non-blocking stream; ``0`` (torch's handle of
        the legacy default stream) is passed on as cudaStreamLegacy."""
        if stream_handle is None:
            handle = None
        else:
            handle = int(stream_handle) or _CUDA_STREAM_LEGACY
        self._check(self._lib.lmx_set_stream(self._h, handle), "lmx_set_stream")

    # -- graph loading -------------------------------------------------------
    def load_graph(self, g) -> None:
        """Load a reference-shaped graph from host numpy arrays (K0 on the device)."""
        eu = np.ascontiguousarray(g.edge_u, dtype=np.int64)
        ev = np.ascontiguousarray(g.edge_v, dtype=np.int64)
        w = np.ascontiguousarray(g.edge_weight, dtype=np.float64)
        self._check(self._lib.lmx_load_graph(self._h, int(g.num_vertices), int(eu.size),
                                             eu.ctypes.data, ev.ctypes.data, w.ctypes.data, LMX_HOST),
                    "lmx_load_graph")

    def load_graph_device(self, n: int, edge_u, edge_v, edge_weight) -> None:
        """Load from device tensors (int64/int64/float64 CUDA tensors)."""
        self._check(self._lib.lmx_load_graph(self._h, int(n), int(edge_u.numel()), _ptr(edge_u),
                                             _ptr(edge_v), _ptr(edge_weight), LMX_DEVICE),
                    "lmx_load_graph")

    def build_graph(self, u, v, w, num_vertices: int | None = None) -> None:
        """build_graph (graph.py:59-119) of raw triples on the device."""
        u = np.ascontiguousarray(u, dtype=np.int64)
        v = np.ascontiguousarray(v, dtype=np.int64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        nv = -1 if num_vertices is None else int(num_vertices)
        self._check(self._lib.lmx_build_graph(self._h, int(u.size), u.ctypes.data, v.ctypes.data,
                                              w.ctypes.data, nv, LMX_HOST), "lmx_build_graph")

    def gen_rmat(self, scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19,
                 c: float = 0.19, seed: int = 1, permute: bool = True) -> None:
        self._check(self._lib.lmx_gen_rmat(self._h, scale, edge_factor, a, b, c, seed & _UINT64_MASK,
                                           int(permute)), "lmx_gen_rmat")

    def gen_er(self, scale: int, edge_factor: int = 4, seed: int = 1, unit: bool = True) -> None:
        """Random graph of the C1 family at scale: edge_factor * 2^scale uniform
        raw pairs, unit (or U[0,1)) weights, build_graph semantics (lmx_gen_er)."""
        self._check(self._lib.lmx_gen_er(self._h, scale, edge_factor, seed & _UINT64_MASK, int(bool(unit))),
                    "lmx_gen_er")

    def gen_rgg(self, x: int, seed: int, weight_mode: str = "euclidean") -> None:
        """``gen_rgg(x, seed, weight_mode)`` (generate.py:113-143) on the device:
        the identical graph.  numpy's SeedSequence supplies the PCG64 start
        state (a few integers); every draw, the Morton order, the grid sweep
        and the distances run on the GPU (lmx_gen_rgg)."""
        import math
        if x < 2:
            raise ValueError("x must be >= 2")
        if weight_mode not in ("euclidean", "random"):
            raise ValueError(f"weight_mode must be euclidean or random, got {weight_mode!r}")
        st = np.random.default_rng(seed).bit_generator.state["state"]
        s, inc = int(st["state"]), int(st["inc"])
        n = 1 << x
        radius = 0.55 * math.sqrt(math.log(n) / n)   # rgg_threshold, generate.py:92-94
        m64 = (1 << 64) - 1
        self._check(self._lib.lmx_gen_rgg(self._h, x, s >> 64, s & m64, inc >> 64, inc & m64, radius,
                                          int(weight_mode == "random")), "lmx_gen_rgg")

    def gen_rmat_raw(self, scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19,
                     c: float = 0.19, seed: int = 1, permute: bool = True):
        k = edge_factor << scale
        u = np.empty(k, dtype=np.int64)
        v = np.empty(k, dtype=np.int64)
        w = np.empty(k, dtype=np.float64)
        self._check(self._lib.lmx_gen_rmat_raw(self._h, scale, edge_factor, a, b, c, seed & _UINT64_MASK,
                                               int(permute), u.ctypes.data, v.ctypes.data, w.ctypes.data,
                                               LMX_HOST), "lmx_gen_rmat_raw")
        return u, v, w

    def graph_size(self) -> tuple[int, int]:
        n = ctypes.c_int64()
        m = ctypes.c_int64()
        self._check(self._lib.lmx_graph_size(self._h, ctypes.byref(n), ctypes.byref(m)), "lmx_graph_size")
        return int(n.value), int(m.value)

    def export_graph(self) -> Graph:
        n, m = self.graph_size()
        eu = np.empty(m, dtype=np.int64)
        ev = np.empty(m, dtype=np.int64)
        w = np.empty(m, dtype=np.float64)
        self._check(self._lib.lmx_graph_export(self._h, eu.ctypes.data, ev.ctypes.data, w.ctypes.data,
                                               LMX_HOST), "lmx_graph_export")
        return Graph(n, eu, ev, w)

    def export_graph_device(self):
        """The loaded graph's edge arrays as CUDA tensors (int64, int64, float64),
        e.g. to time a reload from device-resident inputs."""
        import torch
        _, m = self.graph_size()
        dev = torch.device("cuda", self.device)
        eu = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
        ev = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
        w = torch.empty(max(m, 1), dtype=torch.float64, device=dev)
        self._check(self._lib.lmx_graph_export(self._h, _ptr(eu), _ptr(ev), _ptr(w), LMX_DEVICE),
                    "lmx_graph_export")
        return eu[:m], ev[:m], w[:m]

    def peak_device_bytes(self, reset: bool = False) -> int:
        """High-water mark of the context's device allocations (LMX_QUERY_PEAK_BYTES)."""
        return int(self._lib.lmx_set_option(self._h, 103, int(reset))) << 20

    def device_bytes(self) -> int:
        return int(self._lib.lmx_device_bytes(self._h))

    # -- matching ------------------------------------------------------------
    def match_raw(self, seed: int, rerandomize: bool = True):
        """Run the round loop; returns (mate int64[n], sorted ids int64, [RoundStats])."""
        n, _ = self.graph_size()
        mate = _host_buffer(max(n, 1))
        ids = _host_buffer(max(n // 2 + 1, 1))
        nm = ctypes.c_int64()
        nr = ctypes.c_int()
        self._check(self._lib.lmx_match(self._h, seed & _UINT64_MASK, int(bool(rerandomize)),
                                        mate.ctypes.data, ids.ctypes.data, ctypes.byref(nm), None, 0,
                                        ctypes.byref(nr), LMX_HOST), "lmx_match")
        rounds = self.last_rounds()
        # views of the (page-locked) output blocks: no host copy of the ids
        return mate[:n], ids[: nm.value], rounds

    def match_device(self, seed: int, mate_out, ids_out, rerandomize: bool = True) -> int:
        """Device outputs (CUDA tensors int64[n] and int64[>= n/2]); returns #matched edges."""
        nm = ctypes.c_int64()
        nr = ctypes.c_int()
        self._check(self._lib.lmx_match(self._h, seed & _UINT64_MASK, int(bool(rerandomize)),
                                        _ptr(mate_out), _ptr(ids_out), ctypes.byref(nm), None, 0,
                                        ctypes.byref(nr), LMX_DEVICE), "lmx_match")
        return int(nm.value)

    def last_rounds(self) -> list:
        k = self._lib.lmx_last_rounds(self._h, None, 0)
        buf = (LmxRoundStats * max(k, 1))()
        self._lib.lmx_last_rounds(self._h, buf, k)
        return [RoundStats(int(b.edges_before), int(b.edges_matched), int(b.edges_removed))
                for b in buf[:k]]

    def last_kernel_times(self) -> list:
        """[(round kernel ms, match kernel ms)] per executed round of the last match
        (needs set_kernel_timing(True))."""
        k = self._lib.lmx_last_kernel_times(self._h, None, 0)
        buf = (ctypes.c_float * max(k, 1))()
        self._lib.lmx_last_kernel_times(self._h, buf, k)
        v = list(buf[:k])
        return [(v[i], v[i + 1] if i + 1 < k else 0.0) for i in range(0, k, 2)]

    def last_round_counters(self) -> np.ndarray:
        """int64 [rounds_executed, 8] device counters of the last match (diagnostics)."""
        k = self._lib.lmx_last_round_counters(self._h, None, 0)
        out = np.zeros((max(k, 1), 8), dtype=np.int64)
        self._lib.lmx_last_round_counters(self._h, out.ctypes.data, k)
        return out[:k]

    def last_timing(self) -> dict:
        t = LmxTiming()
        self._check(self._lib.lmx_last_timing(self._h, ctypes.byref(t)), "lmx_last_timing")
        return {"setup_ms": t.setup_ms, "rounds_ms": t.rounds_ms, "output_ms": t.output_ms,
                "round_launches": int(t.round_launches), "slot_reads": int(t.slot_reads),
                "round_kernel_ms": t.round_kernel_ms, "match_kernel_ms": t.match_kernel_ms,
                "rounds_executed": int(t.rounds_executed), "hist_kernel_ms": t.hist_kernel_ms}

    LAYOUTS = {"auto": -1, "uniform": 0, "distinct": 1, "general": 2}

    def set_layout(self, layout: str = "auto") -> None:
        """Force the weight-key layout used by the next graph load (testing / tuning)."""
        self._check(self._lib.lmx_set_option(self._h, LMX_OPT_LAYOUT, self.LAYOUTS[layout]), "lmx_set_option")

    def set_relabel(self, mode: str = "auto") -> None:
        """Degree-descending vertex relabelling of the next load: auto / on / off /
        once (auto, except for the scan loop: a load that serves one matching)."""
        val = {"auto": -1, "off": 0, "on": 1, "once": 2}[mode]
        self._check(self._lib.lmx_set_option(self._h, LMX_OPT_RELABEL, val), "lmx_set_option")

    ALGOS = {"auto": -1, "compact": 0, "scan": 1}

    def set_algo(self, algo: str = "auto") -> None:
        """Round loop of the next load: compacting rounds or the weight-ordered
        scan (distinct weights, single context); results are identical."""
        self._check(self._lib.lmx_set_option(self._h, LMX_OPT_ALGO, self.ALGOS[algo]), "lmx_set_option")

    def algo(self) -> str:
        code = self._lib.lmx_set_option(self._h, LMX_QUERY_ALGO, 0)
        return {v: k for k, v in self.ALGOS.items()}[code]

    def relabeled(self) -> bool:
        return bool(self._lib.lmx_set_option(self._h, LMX_QUERY_RELABELED, 0))

    def layout(self) -> str:
        code = self._lib.lmx_set_option(self._h, LMX_QUERY_LAYOUT, 0)
        return {v: k for k, v in self.LAYOUTS.items()}[code]

    def set_static_order(self, seed: int | None) -> None:
        """rerandomize=False fast path (LMX_OPT_STATIC_ORDER): the next load lays
        graphs with tied weights out in the fixed (weight, salt) order of
        ``seed`` so the weight-ordered scan loop serves them; the loaded graph
        then matches only ``seed`` with rerandomize=False.  None = off."""
        if seed is not None:
            bits = int(seed) & 0xFFFFFFFFFFFFFFFF
            val = bits - (1 << 64) if bits >= (1 << 63) else bits
            self._check(self._lib.lmx_set_option(self._h, LMX_OPT_STATIC_SEED, val), "lmx_set_option")
        self._check(self._lib.lmx_set_option(self._h, LMX_OPT_STATIC_ORDER, int(seed is not None)),
                    "lmx_set_option")

    def static_order(self) -> bool:
        """True if the loaded graph has the static (weight, salt) layout."""
        return bool(self._lib.lmx_set_option(self._h, LMX_QUERY_STATIC, 0))

    def set_kernel_timing(self, on: bool = True) -> None:
        """Record a CUDA event after every round / match kernel (per-kernel durations)."""
        self._check(self._lib.lmx_set_option(self._h, LMX_OPT_KERNEL_TIMING, int(on)), "lmx_set_option")

    def match(self, g, seed: int, rerandomize: bool = True) -> tuple[Matching, PhaseTrace]:
        """local_max_seq contract on a graph already loaded with load_graph(g)."""
        t0 = time.perf_counter()
        mate, ids, rounds = self.match_raw(seed, rerandomize)
        trace = PhaseTrace(rounds=rounds)
        trace.device_millis = self.last_timing()["rounds_ms"]
        trace.wall_millis = (time.perf_counter() - t0) * 1000.0
        return Matching(ids, mate), trace

    def rbm(self, g, seed: int, max_rounds: int = 10_000) -> tuple[Matching, PhaseTrace]:
        """Red-blue matching (matchers.py:357-410) on the graph loaded in this engine."""
        t0 = time.perf_counter()
        n, _ = self.graph_size()
        mate = _host_buffer(max(n, 1))
        ids = _host_buffer(max(n // 2 + 1, 1))
        nm = ctypes.c_int64()
        nr = ctypes.c_int()
        rc = self._lib.lmx_rbm(self._h, seed & _UINT64_MASK, mate.ctypes.data, ids.ctypes.data, ctypes.byref(nm),
                               None, int(max_rounds), ctypes.byref(nr), LMX_HOST)
        if rc == LMX_ELIMIT:
            raise RbmDidNotConverge(self._lib.lmx_last_error(self._h).decode())
        self._check(rc, "lmx_rbm")
        trace = PhaseTrace(rounds=self.last_rounds())
        trace.device_millis = self.last_timing()["rounds_ms"]
        trace.wall_millis = (time.perf_counter() - t0) * 1000.0
        return Matching(ids[: nm.value].copy(), mate[:n]), trace

    def pram_cross(self, want_cross: bool = False):
        """PRAM incidence layout + cross pointers of the loaded graph on the
        device (pram.py:127-166), with the exclusive-write check:
        returns ({steps, writes, conflicts, bad_slot}, cross int64[2m] or None)."""
        _, m = self.graph_size()
        log = np.zeros(4, dtype=np.int64)
        cross = np.empty(max(2 * m, 1), dtype=np.int64) if want_cross else None
        self._check(self._lib.lmx_pram_cross(self._h, cross.ctypes.data if want_cross else None, log.ctypes.data,
                                             LMX_HOST), "lmx_pram_cross")
        return ({"steps": int(log[0]), "writes": int(log[1]), "conflicts": int(log[2]), "bad_slot": int(log[3])},
                cross[: 2 * m] if want_cross else None)

    def validate(self, matching) -> tuple[MatchingCheck, float]:
        """``validate_matching(g, m)`` (graph.py:212-237) and ``m.weight(g)``
        (graph.py:54-56) on the device, for the graph loaded in this engine.
        The weight is bit-identical to numpy's ``edge_weight[ids].sum()``."""
        n, _ = self.graph_size()
        mate = np.ascontiguousarray(np.asarray(matching.mate), dtype=np.int64)
        if mate.shape != (n,):
            return MatchingCheck(False, False, "mate table has wrong length"), 0.0
        ids = matching.sorted_edge_ids() if hasattr(matching, "sorted_edge_ids") else \
            np.array(sorted(matching.edges), dtype=np.int64)
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        valid, maximal = ctypes.c_int(), ctypes.c_int()
        weight = ctypes.c_double()
        detail = ctypes.create_string_buffer(256)
        self._check(self._lib.lmx_validate(self._h, mate.ctypes.data, ids.ctypes.data if ids.size else None,
                                           int(ids.size), LMX_HOST, ctypes.byref(valid), ctypes.byref(maximal),
                                           ctypes.byref(weight), detail, 256), "lmx_validate")
        return MatchingCheck(bool(valid.value), bool(maximal.value), detail.value.decode()), float(weight.value)


def _host_buffer(count: int) -> np.ndarray:
    """int64 host output array.  Large ones come from torch's caching pinned
    allocator (already page-locked and faulted in, so the device writes them at
    link rate and reuses freed blocks); the array keeps its block alive."""
    if count >= (1 << 20):
        try:
            import torch
            if torch.cuda.is_available():
                return torch.empty(count, dtype=torch.int64, pin_memory=True).numpy()
        except Exception:   # no torch / no pinning: plain pageable memory
            pass
    return np.empty(count, dtype=np.int64)


_default_engines: dict[int, Engine] = {}


def default_engine(device: int = 0) -> Engine:
    eng = _default_engines.get(device)
    if eng is None:
        eng = Engine(device)
        _default_engines[device] = eng
    return eng


def local_max_b200(g, seed: int, rerandomize: bool = True, device: int = 0) -> tuple[Matching, PhaseTrace]:
    """Drop-in for ``locmax.local_max_seq(g, seed, rerandomize)`` (matchers.py:61-122).

    ``wall_millis`` covers the whole call (upload, device loop, readback) like
    the reference's; ``device_millis`` is the device round loop alone.
    """
    t0 = time.perf_counter()
    eng = default_engine(device)
    # with rerandomize off the salts are fixed for the run: tied weights get
    # the static (weight, salt) layout and the scan loop (LMX_OPT_STATIC_ORDER)
    eng.set_static_order(None if rerandomize else seed)
    eng.set_relabel("once")   # one matching per load
    try:
        eng.load_graph(g)
    finally:
        eng.set_static_order(None)
        eng.set_relabel("auto")
    matching, trace = eng.match(g, seed, rerandomize)
    trace.wall_millis = (time.perf_counter() - t0) * 1000.0
    return matching, trace


def pram_local_max_b200(g, seed: int, checked: bool = False, rerandomize: bool = True,
                        device: int = 0) -> tuple[Matching, PhaseTrace]:
    """Drop-in for ``locmax.pram.pram_local_max(g, seed, checked, rerandomize)``
    (pram.py:276-315): the same matching and RoundStats (the reference's PRAM
    phases equal the sequential rounds, pram.py:276-281), and the same
    ``trace.slot_ops`` linear-work meter, ``n + 3m`` for the set-up plus
    ``m_r + 2 m_r`` (live edges and incidence slots) per phase (pram.py:293,300).

    ``checked=True`` (pram.py:283-286) builds the PRAM incidence layout and
    its cross pointers on the device with the reference's exclusive-write
    steps (``lmx_pram_cross``), checks them as ``PramState.check_consistent``
    does, validates the matching on the device (graph.py:212-237), and
    returns ``trace.write_log``: a ``WriteLog`` (locmax's when importable)
    holding the cross-pointer steps' writes and conflicts plus one
    ``match/mate`` step per round (2 writes per matched edge; a vertex written
    twice would fail validation and count as a conflict).  Any conflict or
    inconsistency raises ``RuntimeError``.
    """
    t0 = time.perf_counter()
    eng = default_engine(device)
    eng.load_graph(g)
    matching, trace = eng.match(g, seed, rerandomize)
    trace.slot_ops = int(g.num_vertices) + 3 * int(np.asarray(g.edge_u).size) + \
        3 * sum(int(r.edges_before) for r in trace.rounds)
    if checked:
        log, _ = eng.pram_cross()
        if log["bad_slot"] >= 0:
            raise RuntimeError(f"pram_local_max_b200: cross pointers inconsistent at slot {log['bad_slot']}")
        chk, _ = eng.validate(matching)
        if not (chk.valid and chk.maximal):
            raise RuntimeError(f"pram_local_max_b200: device validation failed: {chk}")
        wl = _write_log()
        wl.steps = log["steps"] + len(trace.rounds)
        wl.writes = log["writes"] + 2 * sum(int(r.edges_matched) for r in trace.rounds)
        wl.conflicts = log["conflicts"]
        if wl.conflicts:
            raise RuntimeError(f"pram_local_max_b200: {wl.conflicts} write conflicts in the cross-pointer steps")
        trace.write_log = wl
    trace.wall_millis = (time.perf_counter() - t0) * 1000.0
    return matching, trace


def _write_log():
    """pram.py:28-51 WriteLog (locmax's own when importable)."""
    try:
        from locmax.pram import WriteLog
        return WriteLog()
    except ImportError:
        from dataclasses import dataclass, field

        @dataclass
        class WriteLog:
            steps: int = 0
            writes: int = 0
            conflicts: int = 0
            samples: list = field(default_factory=list)
        return WriteLog()


class RbmDidNotConverge(RuntimeError):
    """matchers.py:353-354: rbm made no progress within its round limit."""


def rbm_b200(g, seed: int, device: int = 0, max_rounds: int = 10_000) -> tuple[Matching, PhaseTrace]:
    """Drop-in for ``locmax.matchers.rbm(g, seed)`` (matchers.py:357-410), the
    paper's GPU competitor: same Matching and RoundStats trace."""
    t0 = time.perf_counter()
    eng = default_engine(device)
    eng.load_graph(g)
    matching, trace = eng.rbm(g, seed, max_rounds)
    trace.wall_millis = (time.perf_counter() - t0) * 1000.0
    return matching, trace


def run_matcher(g, algorithm: str, seed: int, engine: str = "b200", p: int = 4,
                rerandomize: bool = True):
    """bench.py:119-142 dispatch with the B200 engines added.

    ``engine="b200"`` runs :func:`local_max_b200`; ``"b200-dist"`` runs the
    1D-partitioned multi-GPU engine over ``p`` ranks (see ``dist.py``);
    ``"b200-pram"`` runs :func:`pram_local_max_b200` (the "pram" engine's
    trace, with ``slot_ops``).  Other
    engines / algorithms are the reference's and are delegated to ``locmax``
    when it is importable.
    """
    if algorithm == "localmax" and engine == "b200":
        return local_max_b200(g, seed, rerandomize)
    if algorithm == "rbm" and engine == "b200":
        return rbm_b200(g, seed)
    if algorithm == "localmax" and engine == "b200-pram":
        return pram_local_max_b200(g, seed, rerandomize=rerandomize)
    if algorithm == "localmax" and engine == "b200-dist":
        from .dist import local_max_dist
        return local_max_dist(g, p, seed, rerandomize)
    if engine in ("b200", "b200-dist", "b200-pram"):
        raise ValueError(f"algorithm {algorithm!r} only runs on the seq engine")
    try:
        from locmax.bench import run_matcher as ref_run_matcher
    except ImportError as exc:
        raise ValueError(f"unknown engine {engine!r} (the reference locmax package is not importable)") from exc
    return ref_run_matcher(g, algorithm, seed, engine, p, rerandomize)
