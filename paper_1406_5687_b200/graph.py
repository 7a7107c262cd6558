"""Degree-ordered graph container on the device (mirrors graph.py:1-160 of
the reference `tricount`).

Canonical ids order nodes by ascending (degree, original id); every edge is
stored once on the forward list N^_v of its lower endpoint.  Construction
runs entirely on the GPU (csrc/build.cu): device radix sorts give exactly
numpy's stable lexsort / unique orderings, so relabel, orig_ids and the CSR
arrays are bit-identical to the reference's.

Layout (HBM): node ids int32, CSR offsets int64 (the reference uses int64
everywhere).  Besides the reference's fields the Graph keeps the reverse
("predecessor") CSR the middle-vertex engine streams: for every oriented edge
(v, u) the suffix of N^_v after u, grouped by u.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib

_I32_MAX = 2**31 - 1
POOL_HEAD = 512  # TC_POOL_HEAD (include/tcb200.h)


def _as_device_pairs(edges, dev):
    """(m, 2) int32 contiguous device tensor from any array-like of pairs."""
    if isinstance(edges, torch.Tensor):
        t = edges.reshape(-1, 2)
        if t.dtype != torch.int32:
            if t.numel():
                lo, hi = torch.aminmax(t)
                # checked before the cast: an int64 label below -2^31 would wrap
                # to a non-negative int32 id (graph.py:87-88 rejects negatives)
                if int(lo) < 0:
                    raise ValueError("negative node id in edge list")
                if int(hi) > _I32_MAX:
                    raise ValueError("node labels must fit int32 on the B200 path")
            t = t.to(torch.int32)
        return t.to(dev, non_blocking=True).contiguous()
    a = np.asarray(edges)
    if a.size == 0:
        return torch.empty((0, 2), dtype=torch.int32, device=dev)
    a = a.reshape(-1, 2)
    if a.dtype != np.int32:
        if int(a.max()) > _I32_MAX:
            raise ValueError("node labels must fit int32 on the B200 path")
        if int(a.min()) < -(2**31):
            raise ValueError("negative node id in edge list")
        a = a.astype(np.int32)
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev, non_blocking=True)


@dataclass(frozen=True)
class RawGraph:
    """Edge list before normalization (graph.py:17-33).

    `n` is the declared node count; `edges` is an (m, 2) array of undirected
    pairs (numpy, list or torch tensor; host or device) with non-negative
    labels that fit int32.
    """

    n: int
    edges: object
    # degree of every node of a normalized list, when normalize computed it
    # on the way (host-input pipeline); build_graph then skips its histogram
    _deg: object = field(default=None, repr=False, compare=False)

    @classmethod
    def from_pairs(cls, pairs, n=None):
        edges = np.asarray(list(pairs), dtype=np.int64).reshape(-1, 2)
        if n is None:
            n = int(edges.max()) + 1 if edges.size else 0
        return cls(n=n, edges=edges)

    def device_edges(self):
        return _as_device_pairs(self.edges, _lib.device())


class Graph:
    """Immutable degree-ordered graph with CSR adjacency on the device
    (graph.py:36-73).  Array fields are torch tensors on the GPU."""

    __slots__ = ("n", "m", "eff_indptr", "eff_indices", "relabel", "orig_ids", "deg", "eff_deg",
                 "_rev_indptr", "_rev_seg", "_rev_cost", "_pool_indptr", "_pool", "_full", "_cache")

    def __init__(self, n, m, eff_indptr, eff_indices, relabel, orig_ids, deg, eff_deg, rev_indptr,
                 rev_seg, rev_cost, pool_indptr, pool):
        self.n, self.m = int(n), int(m)
        self.eff_indptr, self.eff_indices = eff_indptr, eff_indices
        self.relabel, self.orig_ids, self.deg, self.eff_deg = relabel, orig_ids, deg, eff_deg
        # reverse CSR for the pull engine: per u, the (start, end) int32 pairs of
        # its predecessors' suffixes in _pool coordinates (rows unordered)
        self._rev_indptr, self._rev_seg, self._rev_cost = rev_indptr, rev_seg, rev_cost
        # the engine's row-padded copy of the forward lists (rows at multiples
        # of 4 ids, INT32_MAX padding, POOL_HEAD INT32_MAX ids before _pool[0]);
        # rev_seg's coordinates index it
        self._pool_indptr, self._pool = pool_indptr, pool
        self._full = None
        self._cache = {}

    # -- full CSR (graph.py:125-127), assembled lazily on the device ---------
    def _full_csr(self):
        if self._full is None:
            dev = self.eff_indptr.device
            fip = torch.empty(self.n + 1, dtype=torch.int64, device=dev)
            fix = torch.empty(max(2 * self.m, 1), dtype=torch.int32, device=dev)
            _lib.call("tc_build_full", _lib.ptr(self.eff_indptr), _lib.ptr(self.eff_indices),
                      _lib.ptr(self._rev_indptr), _lib.ptr(self._rev_seg), _lib.ptr(self._pool_indptr), self.n,
                      _lib.ptr(fip),
                      _lib.ptr(fix), _lib.stream())
            self._full = (fip, fix[: 2 * self.m])
        return self._full

    @property
    def full_indptr(self):
        return self._full_csr()[0]

    @property
    def full_indices(self):
        return self._full_csr()[1]

    def neighbors(self, v):
        """All neighbors of canonical node v, ascending."""
        ip = self.full_indptr
        return self.full_indices[int(ip[v]): int(ip[v + 1])]

    def succ(self, v):
        """Higher-ordered neighbors of canonical node v, ascending."""
        return self.eff_indices[int(self.eff_indptr[v]): int(self.eff_indptr[v + 1])]

    def precedes(self, u, v):
        """Whether u comes strictly before v in the counting order (graph.py:64-68)."""
        if not (0 <= u < self.n and 0 <= v < self.n):
            raise IndexError(f"node id out of range: ({u}, {v}) with n={self.n}")
        return u < v

    def canonical_edges(self):
        """(m, 2) tensor of (low, high) canonical pairs, sorted (graph.py:70-73)."""
        src = torch.repeat_interleave(torch.arange(self.n, dtype=torch.int32, device=self.eff_indices.device),
                                      self.eff_deg.to(torch.int64), output_size=self.m)
        return torch.stack([src, self.eff_indices], dim=1)

    def to_host(self):
        """numpy copies of the reference's fields (int64, like the reference)."""
        f = lambda t: t.detach().cpu().numpy().astype(np.int64)  # noqa: E731
        return dict(n=self.n, m=self.m, eff_indptr=f(self.eff_indptr), eff_indices=f(self.eff_indices),
                    full_indptr=f(self.full_indptr), full_indices=f(self.full_indices),
                    relabel=f(self.relabel), orig_ids=f(self.orig_ids), deg=f(self.deg),
                    eff_deg=f(self.eff_deg))


# List entries per L2 tile of the optional tiled predecessor index (0 = off).
TILE_IDS = int(os.environ.get("TCB_TILE_IDS", "0"))


@dataclass
class TiledIndex:
    """Predecessor entries of u in [u0, u1) regrouped tile-major (csrc/tile.cu)."""

    u0: int
    u1: int
    k: int
    ntiles: int
    owner_u: torch.Tensor
    owner_ptr: torch.Tensor
    segs: torch.Tensor
    cost: torch.Tensor


def tiled_index(g: "Graph", u0: int, u1: int) -> TiledIndex:
    key = ("tiled", u0, u1, TILE_IDS)
    t = g._cache.get(key)
    if t is None:
        dev = g.eff_indptr.device
        E = int(g._rev_indptr[u1] - g._rev_indptr[u0]) if g.n else 0
        owner_u = torch.empty(max(E, 1), dtype=torch.int32, device=dev)
        owner_ptr = torch.empty(E + 1, dtype=torch.int64, device=dev)
        segs = torch.empty(max(2 * E, 2), dtype=torch.int32, device=dev)
        cost = torch.empty(E + 1, dtype=torch.int64, device=dev)
        k, nt = ctypes.c_int64(), ctypes.c_int64()
        if g.n:
            _lib.call("tc_tile_pull", _lib.ptr(g.eff_indptr), _lib.ptr(g._pool_indptr), g.n, _lib.ptr(g._rev_indptr),
                      _lib.ptr(g._rev_seg), u0, u1, TILE_IDS, _lib.ptr(owner_u), _lib.ptr(owner_ptr),
                      _lib.ptr(segs), _lib.ptr(cost), ctypes.byref(k), ctypes.byref(nt), _lib.stream())
        else:
            owner_ptr.zero_()
            cost.zero_()
        t = TiledIndex(u0, u1, k.value, nt.value, owner_u, owner_ptr, segs, cost)
        g._cache[key] = t
    return t


def normalize(raw: RawGraph) -> RawGraph:
    """Drop self-loops, collapse duplicate undirected edges and compact labels
    to 0..n-1 (graph.py:76-103), on the device.  Dense labels are kept as-is;
    sparse labels get compact ids in first-seen order of the raveled edge
    list.  Returns a RawGraph whose edges are a sorted (m, 2) int32 device
    tensor."""
    dev = _lib.device()
    h = raw.edges
    if (isinstance(h, torch.Tensor) and h.device.type == "cpu" and h.dtype == torch.int32 and h.is_pinned()
            and h.is_contiguous() and h.numel() >= _HOST_PIPELINE_MIN):
        return _normalize_host(h.reshape(-1, 2), dev)
    e = _as_device_pairs(raw.edges, dev)
    m_raw = e.shape[0]
    out = torch.empty((max(m_raw, 1), 2), dtype=torch.int32, device=dev)
    m = ctypes.c_int64(0)
    n = ctypes.c_int64(0)
    _lib.call("tc_normalize", _lib.ptr(e), m_raw, _lib.ptr(out), ctypes.byref(m), ctypes.byref(n),
              _lib.stream())
    return RawGraph(n=int(n.value), edges=out[: m.value])


# host lists of at least this many ids take the chunked copy pipeline
_HOST_PIPELINE_MIN = int(os.environ.get("TCB_HOST_PIPELINE_MIN", 1 << 23))


def _normalize_host(h, dev) -> RawGraph:
    """normalize of a pinned host int32 list: the H2D copy runs in chunks on a
    copy stream with each chunk's first-occurrence / degree passes behind it
    (tc_normalize_host)."""
    m_raw = h.shape[0]
    staging = torch.empty((m_raw, 2), dtype=torch.int32, device=dev)
    out = torch.empty((m_raw, 2), dtype=torch.int32, device=dev)
    deg = torch.empty(2 * m_raw + 1, dtype=torch.int32, device=dev)
    m, n, valid = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int32(0)
    _lib.call("tc_normalize_host", _lib.ptr(h), m_raw, _lib.ptr(staging), _lib.ptr(out), ctypes.byref(m),
              ctypes.byref(n), _lib.ptr(deg), ctypes.byref(valid), _lib.stream())
    del staging
    nv = int(n.value)
    return RawGraph(n=nv, edges=out[: m.value], _deg=deg[:nv] if valid.value else None)


def _assemble(raw: RawGraph, order) -> Graph:
    dev = _lib.device()
    e = _as_device_pairs(raw.edges, dev)
    n, m = int(raw.n), int(e.shape[0])
    i64 = lambda k: torch.empty(max(k, 1), dtype=torch.int64, device=dev)  # noqa: E731
    i32 = lambda k: torch.empty(max(k, 1), dtype=torch.int32, device=dev)  # noqa: E731
    # +4 ids of padding: the engines read lists as 16-byte chunks
    eff_indptr, eff_indices = i64(n + 1), i32(m + 4)
    relabel, orig_ids, deg, eff_deg = i32(n), i32(n), i32(n), i32(n)
    rev_indptr, rev_seg, rev_cost = i64(n + 1), i32(2 * m), i64(n + 1)
    pool_indptr = i64(n + 1)
    pool_buf = i32(POOL_HEAD + m + 3 * n + 4)  # +4: never an empty view (data_ptr would be NULL)
    pool = pool_buf[POOL_HEAD:]
    order_t = None
    if order is not None:
        order_t = torch.as_tensor(np.asarray(order, dtype=np.int32)).to(dev).contiguous()
    hint = raw._deg if (order is None and raw._deg is not None and raw._deg.numel() == n) else None
    _lib.call("tc_build_graph" if hint is None else "tc_build_graph_deg", _lib.ptr(e), m, n,
              _lib.ptr(order_t if hint is None else hint), _lib.ptr(eff_indptr),
              _lib.ptr(eff_indices), _lib.ptr(relabel), _lib.ptr(orig_ids), _lib.ptr(deg),
              _lib.ptr(eff_deg), _lib.ptr(rev_indptr), _lib.ptr(rev_seg), _lib.ptr(rev_cost), _lib.ptr(pool_indptr),
              _lib.ptr(pool), _lib.stream())
    g = Graph(n, m, eff_indptr[: n + 1], eff_indices[:m], relabel[:n], orig_ids[:n], deg[:n],
              eff_deg[:n], rev_indptr[: n + 1], rev_seg[: 2 * m], rev_cost[: n + 1], pool_indptr[: n + 1], pool)
    if TILE_IDS:
        tiled_index(g, 0, n)  # optional L2-tiled predecessor index, built with the graph
    return g


def build_graph(raw: RawGraph) -> Graph:
    """Relabel a normalized RawGraph into degree order and build adjacency
    (graph.py:143-153): ascending (degree, original id), each edge stored once
    on its lower endpoint's forward list.  Like the reference it does not
    deduplicate; declared isolated nodes (raw.n) are kept."""
    return _assemble(raw, None)


def _build_graph_input_order(raw: RawGraph) -> Graph:
    """Test hook: identity relabeling (graph.py:156-160)."""
    return _assemble(raw, np.arange(raw.n, dtype=np.int32))
