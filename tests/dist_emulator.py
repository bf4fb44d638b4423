"""CPU emulation of one liblmx distributed partition -- TEST INFRASTRUCTURE ONLY.

Implements the per-rank interface ``paper_1302_4587_b200.dist.run_rounds``
drives (begin / round / propose / recv_buffer / accept / match, plus the
``bitmap`` / ``mate`` / ``ebits`` tensors and ``word_range``), restating the
device kernels' semantics in numpy on CPU tensors.  It exists so the
multi-process transport (``TorchComm`` over gloo, world_size 2) and the
round protocol can be tested on a machine without a GPU.  The product path
never uses it.
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import oracle as O


def partition_bounds(n: int, eu, ev, p: int) -> np.ndarray:
    """partition_graph's cut rule (bsp.py:60-98), as csrc/lmx_setup.cu:partition_bounds."""
    deg = np.bincount(np.concatenate([eu, ev]), minlength=n).astype(np.int64)
    offsets = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    return O.partition_bounds(offsets, n, p)


class EmulatedRank:
    """``algo`` mirrors the device loop the partition emulates: "compact"
    (match reports live slots) or "scan" (match reports candidates found;
    ``mround`` + ``hist`` give the statistics after the loop)."""

    def __init__(self, g, p: int, rank: int, algo: str = "compact"):
        self.p, self.rank, self.algo = p, rank, algo
        self.device = torch.device("cpu")
        self.n, self.m = int(g.num_vertices), int(np.asarray(g.edge_u).size)
        self.eu = np.asarray(g.edge_u, dtype=np.int64)
        self.ev = np.asarray(g.edge_v, dtype=np.int64)
        self.wb = O.weight_bits(np.asarray(g.edge_weight, dtype=np.float64))
        self.bounds = partition_bounds(self.n, self.eu, self.ev, p)
        self.lo, self.hi = int(self.bounds[rank]), int(self.bounds[rank + 1])
        self.words = (self.n + 31) // 32
        self.bitmap = torch.zeros(max(self.words, 1), dtype=torch.int32)
        self.mate = torch.full((max(self.n, 1),), -1, dtype=torch.int64)
        self.ebits = torch.zeros((max(self.m, 1) + 31) // 32, dtype=torch.int32)
        self.mround = torch.full((max(self.n, 1),), -1, dtype=torch.int32) if (algo == "scan" or p > 1) else None

    def vertex_range(self, k: int):
        return int(self.bounds[k]), int(self.bounds[k + 1])

    def hist(self, n_rounds: int):
        """Death rounds of the edges whose higher end this partition owns."""
        mr = self.mround.numpy().view(np.uint32).astype(np.int64)
        hi = np.maximum(self.eu, self.ev)
        own = (hi >= self.lo) & (hi < self.hi)
        d = np.minimum(np.minimum(mr[self.eu[own]], mr[self.ev[own]]), n_rounds)
        return torch.from_numpy(np.bincount(d, minlength=max(n_rounds + 1, 256)).astype(np.int64))

    def messages(self, n_rounds: int):
        """lmx_dist_messages restated: candidate records by the last round
        they are sent in (per owned vertex, its end of the edge and the
        receiving partition: bsp.py:152-154 dedupes the edge_u and edge_v sides
        separately) and cut edges by death round (each once, from its lower end)."""
        mr = self.mround.numpy().view(np.uint32).astype(np.int64)
        rec = np.zeros(n_rounds + 1, dtype=np.int64)
        cut = np.zeros(n_rounds + 1, dtype=np.int64)
        ou = np.searchsorted(self.bounds, self.eu, side="right") - 1
        ov = np.searchsorted(self.bounds, self.ev, side="right") - 1
        death = np.minimum(np.minimum(mr[self.eu], mr[self.ev]), n_rounds)
        best = {}   # (vertex, its end of the edge (0 = edge_u, 1 = edge_v), receiving worker) -> last round
        for e in np.nonzero(ou != ov)[0]:
            for end, x, wx, y, wy in ((0, self.eu[e], ou[e], self.ev[e], ov[e]), (1, self.ev[e], ov[e], self.eu[e], ou[e])):
                if wx != self.rank:
                    continue
                key = (int(x), end, int(wy))
                best[key] = max(best.get(key, -1), int(death[e]))
                if x < y:
                    cut[death[e]] += 1
        for d in best.values():
            rec[d] += 1
        return torch.from_numpy(np.concatenate([rec, cut]))

    def word_range(self, k: int):
        # the bitmap words holding range k's bits (boundary words are shared)
        return int(self.bounds[k]) // 32, (int(self.bounds[k + 1]) + 31) // 32

    def _owner(self, x: int) -> int:
        return int(np.searchsorted(self.bounds, x, side="right") - 1)

    def _is_matched(self, v: int) -> bool:
        w = int(self.bitmap[v >> 5].item()) & 0xFFFFFFFF
        return bool((w >> (v & 31)) & 1)

    def begin(self, seed: int, rerandomize: bool):
        self.seed, self.rr, self.r = seed, rerandomize, 0
        self.adj = {}
        for e in range(self.m):
            for a, b in ((self.eu[e], self.ev[e]), (self.ev[e], self.eu[e])):
                if self.lo <= a < self.hi:
                    self.adj.setdefault(int(a), []).append((int(b), e))
        self.bitmap.zero_()
        self.mate.fill_(-1)
        self.ebits.zero_()
        self.cand = {}
        self.remote_ok = set()
        if self.mround is not None:
            self.mround.fill_(-1)

    def round(self):
        rs = O.round_seed(self.seed, self.r, self.rr)
        self.cand = {}
        self.live_slots = 0
        for v, lst in self.adj.items():
            if self._is_matched(v):
                continue
            lst = [(x, e) for (x, e) in lst if not self._is_matched(x)]
            self.adj[v] = lst
            self.live_slots += len(lst)
            if lst:
                best = max(lst, key=lambda t: (int(self.wb[t[1]]), int(O.edge_salts(rs, [t[1]])[0])))
                self.cand[v] = best

    def propose(self):
        groups = [[] for _ in range(self.p)]
        for v, (x, e) in self.cand.items():
            if not (self.lo <= x < self.hi):
                groups[self._owner(x)].append((x, e))
        counts = torch.tensor([len(gp) for gp in groups], dtype=torch.int64)
        self._groups = groups
        flat = [rec for gp in groups for rec in gp]
        send = torch.tensor(flat if flat else np.zeros((0, 2)), dtype=torch.int32).reshape(-1, 2)
        return send, counts

    def pad(self, capacity: int):
        """lmx_dist_pad restated: p slots of `capacity` records, filler
        {first vertex of the slot's owner, kNone} after each slot's records."""
        C = int(capacity)
        out = np.zeros((self.p * C, 2), dtype=np.int64)
        overflow = 0
        for j, gp in enumerate(self._groups):
            overflow |= int(len(gp) > C)
            for t in range(C):
                out[j * C + t] = gp[t] if t < len(gp) else (int(self.bounds[j]), 0xFFFFFFFF)
        return (torch.from_numpy(out.astype(np.uint32).view(np.int32)).reshape(-1, 2),
                torch.tensor([overflow], dtype=torch.int32))

    def list_size(self):
        """A_{r+1}: the owned vertices that found a candidate and stayed unmatched."""
        return torch.tensor([sum(1 for v in self.cand if not self._is_matched(v))], dtype=torch.int32)

    def recv_buffer(self, count: int):
        self.recv = torch.zeros((int(count), 2), dtype=torch.int32)
        return self.recv

    def accept(self, count: int):
        self.remote_ok = set()
        for x, e in self.recv[: int(count)].tolist():
            if x in self.cand and self.cand[x][1] == e:
                self.remote_ok.add(x)

    def match(self):
        mv = 0
        words = self.bitmap.numpy().view(np.uint32)
        eb = self.ebits.numpy().view(np.uint32)
        for v, (x, e) in self.cand.items():
            if self.lo <= x < self.hi:
                mutual = x in self.cand and self.cand[x][1] == e
            else:
                mutual = v in self.remote_ok
            if mutual:
                words[v >> 5] |= np.uint32(1 << (v & 31))
                self.mate[v] = x
                if self.mround is not None:
                    self.mround[v] = self.r
                mv += 1
                if v < x:
                    eb[e >> 5] |= np.uint32(1 << (e & 31))
        self.r += 1
        first = len(self.cand) if self.algo == "scan" else self.live_slots
        return torch.tensor([first, mv], dtype=torch.int64)
