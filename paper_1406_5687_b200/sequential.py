"""Exact triangle counting on one GPU (mirrors sequential.py:1-51).

count_triangles_seq runs the middle-vertex engine (csrc/count.cu) over the
whole graph; every triangle v < u < w is found exactly once, at its middle
vertex u, so the total equals the reference's lowest-vertex sum
(count_node_range(0, n), _kernels.py:40-52).  The brute-force counter is a
separate dense-bitmap kernel that shares no code with the engines.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .graph import Graph, tiled_index

BRUTE_MAX_NODES = 2000


def _dev_list(a, dev):
    if isinstance(a, torch.Tensor):
        return a.to(dev, torch.int32).contiguous()
    return torch.as_tensor(np.asarray(a, dtype=np.int64).astype(np.int32)).to(dev)


def intersect_count(a, b) -> int:
    """Size of the intersection of two strictly ascending id lists
    (sequential.py:20-27)."""
    dev = _lib.device()
    a, b = _dev_list(a, dev), _dev_list(b, dev)
    if __debug__:
        assert a.numel() < 2 or bool((a[1:] > a[:-1]).all()), "first list not ascending"
        assert b.numel() < 2 or bool((b[1:] > b[:-1]).all()), "second list not ascending"
    out = torch.empty(1, dtype=torch.int64, device=dev)
    _lib.call("tc_intersect_count", _lib.ptr(a), a.numel(), _lib.ptr(b), b.numel(), _lib.ptr(out),
              _lib.stream())
    return int(out.item())


class _MiddlePlan:
    """Owner of a tc_plan_t (tier lists + chunk plan of one (graph, range)),
    cached on the Graph; freed with it."""

    __slots__ = ("handle",)

    def __init__(self, g: Graph, u0: int, u1: int, parts: int = 1):
        import ctypes

        h = ctypes.c_void_p()
        _lib.call("tc_plan_middle_parts", _lib.ptr(g.eff_indptr), _lib.ptr(g.eff_indices), _lib.ptr(g._rev_indptr),
                  _lib.ptr(g._rev_seg), _lib.ptr(g._rev_cost), _lib.ptr(g._pool), 1, g.n, u0, u1, None, 1,
                  int(parts), ctypes.byref(h), _lib.stream())
        self.handle = h

    def run(self, out, part=-1):
        _lib.call("tc_plan_run_part", self.handle, int(part), _lib.ptr(out), _lib.stream())

    def __del__(self):
        try:
            if self.handle:
                _lib.lib().tc_plan_free(self.handle)
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass


def count_middle(g: Graph, u0=0, u1=None, bounds=None, out=None, tiled=None):
    """Middle-vertex engine over u in [u0, u1), optionally binned by `bounds`
    (device int64[k+1]).  Returns the device uint64 counts (as int64).

    tiled=True runs over the L2-tiled predecessor index of the range
    (graph.tiled_index, cached on the graph); the default follows
    TCB_TILE_IDS (off unless set)."""
    u1 = g.n if u1 is None else u1
    if tiled is None:
        from .graph import TILE_IDS
        tiled = TILE_IDS > 0
    k = 1 if bounds is None else int(bounds.numel()) - 1
    if out is None:
        out = torch.empty(k, dtype=torch.int64, device=g.eff_indptr.device)
    if tiled:
        t = tiled_index(g, int(u0), int(u1))
        _lib.call("tc_count_owners", _lib.ptr(g.eff_indptr), _lib.ptr(g.eff_indices), _lib.ptr(t.owner_u),
                  _lib.ptr(t.owner_ptr), _lib.ptr(t.segs), _lib.ptr(t.cost), _lib.ptr(g._pool), t.k,
                  _lib.ptr(bounds), k, _lib.ptr(out), 1, _lib.stream())
        return out
    if bounds is None:  # repeated counts of one graph reuse the engine plan
        key = ("middle_plan", int(u0), int(u1))
        plan = g._cache.get(key)
        if plan is None:
            plan = g._cache[key] = _MiddlePlan(g, int(u0), int(u1))
        plan.run(out)
        return out
    _lib.call("tc_count_middle", _lib.ptr(g.eff_indptr), _lib.ptr(g.eff_indices),
              _lib.ptr(g._rev_indptr), _lib.ptr(g._rev_seg), _lib.ptr(g._rev_cost),
              _lib.ptr(g._pool), 1, g.n, int(u0), int(u1), _lib.ptr(bounds), k, _lib.ptr(out),
              _lib.stream())
    return out


def count_middle_part(g: Graph, part: int, parts: int, out=None):
    """The chunks c with c mod parts == part of the whole-graph middle-vertex
    engine plan, cut for `parts` devices (tc_plan_middle_parts): the
    replicated multi-GPU count, where every rank holds the graph and the
    rank partials sum (NCCL all-reduce) to the total.  Every tier is split
    between the parts, so they stay balanced whatever the cost model's
    error between tiers (dynamic_lb.py:68-109 across ranks)."""
    if not 0 <= part < parts:
        raise ValueError("part must be in [0, parts)")
    if out is None:
        out = torch.empty(1, dtype=torch.int64, device=g.eff_indptr.device)
    key = ("middle_plan_parts", int(parts))
    plan = g._cache.get(key)
    if plan is None:
        plan = g._cache[key] = _MiddlePlan(g, 0, g.n, parts)
    plan.run(out, part)
    return out


def count_lowest(g: Graph, v0=0, v1=None, bounds=None, out=None):
    """Lowest-vertex engine: count_node_range(v0, v1) (_kernels.py:40-52),
    optionally binned by `bounds` (device int64[k+1])."""
    v1 = g.n if v1 is None else v1
    k = 1 if bounds is None else int(bounds.numel()) - 1
    if out is None:
        out = torch.empty(k, dtype=torch.int64, device=g.eff_indptr.device)
    _lib.call("tc_count_lowest", _lib.ptr(g.eff_indptr), _lib.ptr(g.eff_indices), g.n, int(v0),
              int(v1), _lib.ptr(bounds), k, _lib.ptr(out), _lib.stream())
    return out


def count_merge_path(g: Graph, out=None):
    """count_node_range(0, n) by warp-per-edge merge-path / binary-search
    intersections (merge_count per oriented edge, _kernels.py:15-52): the
    formulation the north star names, kept as the measured comparator of
    the middle-vertex engine."""
    if out is None:
        out = torch.empty(1, dtype=torch.int64, device=g.eff_indptr.device)
    _lib.call("tc_count_merge_path", _lib.ptr(g.eff_indptr), _lib.ptr(g.eff_indices), g.n, _lib.ptr(out),
              _lib.stream())
    return out


def count_triangles_seq(g: Graph) -> int:
    """Exact triangle count of g (sequential.py:30-34)."""
    if g.n < 3:
        return 0
    return int(count_middle(g).item())


def count_triangles_brute(g: Graph) -> int:
    """Exact count from a dense adjacency bitmap; oracle-style, n <= 2000
    (sequential.py:37-51)."""
    if g.n > BRUTE_MAX_NODES:
        raise ValueError(f"brute-force counter limited to n <= {BRUTE_MAX_NODES}")
    if g.n < 3:
        return 0
    out = torch.empty(1, dtype=torch.int64, device=g.eff_indptr.device)
    _lib.call("tc_count_brute", _lib.ptr(g.full_indptr), _lib.ptr(g.full_indices), g.n, _lib.ptr(out),
              _lib.stream())
    return int(out.item())
