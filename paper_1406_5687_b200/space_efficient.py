"""Counting over non-overlapping node-range partitions with the surrogate
and the direct schemes (mirrors space_efficient.py:1-262 of the reference).

Each rank owns the forward lists of one consecutive, cost-balanced node
range (PRED_SUM by default, partitioning.py:139-141).  For an oriented edge
(v, u) with u owned elsewhere, v's owner ships N^_v once to u's owner
(LastProc dedup) and the receiver counts
|N^_u ∩ N^_v| for its own u.  Per-rank partials are therefore the triangles
whose MIDDLE vertex the rank owns -- exactly what the middle-vertex engine
computes when binned by the rank bounds, so on one device the partials and
the message census come from two kernels.  The multi-GPU execution (real
exchange over NCCL) is in distributed.py.
"""

from __future__ import annotations

import ctypes
import time

import numpy as np
import torch

from . import _lib
from .graph import Graph
from .partitioning import CostKind, NodeRange, partition_ranges, range_bounds
from .results import WORD_BYTES, RankMetrics, RunResult
from .sequential import count_lowest, count_middle

SCAN_CHUNK = 256  # reference constant (space_efficient.py:43); the device scan has no chunking


def dedup_send_targets(neighbors, bounds, self_rank=-1):
    """Ranks owning at least one id of an ascending list, in first-occurrence
    order, excluding self_rank (space_efficient.py:46-63)."""
    nb = np.asarray(neighbors.cpu() if isinstance(neighbors, torch.Tensor) else neighbors, dtype=np.int64)
    if nb.size == 0:
        return []
    owners = np.searchsorted(np.asarray(bounds, dtype=np.int64), nb, side="right") - 1
    out = []
    last = -1
    for j in owners.tolist():
        if j != self_rank and j != last:
            out.append(j)
            last = j
    return out


def surrogate_count(x, core: NodeRange, g: Graph) -> int:
    """Triangles found by scanning a received neighbor list x against the
    lists of x's members inside `core` (space_efficient.py:66-74;
    _kernels.py:70-80), on the device via the middle-vertex engine."""
    dev = g.eff_indptr.device
    xh = np.asarray(x.cpu() if isinstance(x, torch.Tensor) else x, dtype=np.int64).astype(np.int32)
    if xh.size == 0 or core.count == 0:
        return 0
    buf = torch.zeros(xh.size + 4, dtype=torch.int32, device=dev)  # padded for 16-byte chunk reads
    buf[: xh.size] = torch.as_tensor(xh).to(dev)
    xs = buf[: xh.size]
    offs = torch.tensor([0, xs.numel()], dtype=torch.int64, device=dev)
    segs_owner, segs, nseg = owner_segments(offs, xs, core.start, core.stop, 0)
    return count_segments(g.eff_indptr[core.start:], g.eff_indices, xs, segs_owner, segs, nseg,
                          core.count)


def owner_segments(list_offsets, list_ids, lo, hi, pool_base):
    """Device segments (owner, suffix) for owned ids found in the lists."""
    nl = int(list_offsets.numel()) - 1
    cnt = ctypes.c_int64()
    cap = max(int(list_ids.numel()), 1)  # at most one segment per id
    dev = list_ids.device
    owner = torch.empty(cap, dtype=torch.int32, device=dev)
    segs = torch.empty(2 * cap, dtype=torch.int32, device=dev)
    _lib.call("tc_owner_segments", _lib.ptr(list_offsets), _lib.ptr(list_ids), nl, int(lo), int(hi),
              int(pool_base), _lib.ptr(owner), _lib.ptr(segs), cap, ctypes.byref(cnt), _lib.stream())
    return owner, segs, cnt.value


def segments_csr(owner, segs, nseg, n_owner, tab_indptr):
    """Segments grouped by owner: (row_indptr, row_segs, cost_prefix) for the
    middle-vertex engine (tables tab_indptr indexed 0..n_owner)."""
    dev = segs.device
    row = torch.empty(n_owner + 1, dtype=torch.int64, device=dev)
    rsegs = torch.empty(max(2 * nseg, 2), dtype=torch.int32, device=dev)
    cost = torch.empty(n_owner + 1, dtype=torch.int64, device=dev)
    _lib.call("tc_segments_csr", _lib.ptr(owner), _lib.ptr(segs), int(nseg), int(n_owner),
              _lib.ptr(tab_indptr.contiguous()), _lib.ptr(row), _lib.ptr(rsegs), _lib.ptr(cost), _lib.stream())
    return row, rsegs, cost


def count_segments(tab_indptr, tab_indices, pool, owner, segs, nseg, n_owner, bounds=None):
    """Middle-vertex engine over explicit segments (tables indexed 0..n_owner)."""
    dev = pool.device
    tab_indptr = tab_indptr.contiguous()
    row, rsegs, cost = segments_csr(owner, segs, nseg, n_owner, tab_indptr)
    k = 1 if bounds is None else int(bounds.numel()) - 1
    out = torch.empty(k, dtype=torch.int64, device=dev)
    _lib.call("tc_count_middle", _lib.ptr(tab_indptr), _lib.ptr(tab_indices), _lib.ptr(row),
              _lib.ptr(rsegs), _lib.ptr(cost), _lib.ptr(pool), 0, int(n_owner), 0, int(n_owner),
              _lib.ptr(bounds), k, _lib.ptr(out), _lib.stream())
    return int(out.sum().item()) if bounds is None else out


def surrogate_census(g: Graph, bounds_dev, P):
    """(census[P,P], words[P]) of the LastProc records (_kernels.py:94-126)."""
    dev = g.eff_indptr.device
    census = torch.empty(P * P, dtype=torch.int64, device=dev)
    words = torch.empty(P, dtype=torch.int64, device=dev)
    _lib.call("tc_surrogate_census", _lib.ptr(g.eff_indptr), _lib.ptr(g.eff_indices), g.n,
              _lib.ptr(bounds_dev), int(P), _lib.ptr(census), _lib.ptr(words), _lib.stream())
    return census.view(P, P).cpu().numpy(), words.cpu().numpy()


def _partition_bytes(eff_indptr_h, lo, hi):
    return WORD_BYTES * ((hi - lo) + 1 + int(eff_indptr_h[hi] - eff_indptr_h[lo]))


def count_space_surrogate(g: Graph, nranks: int, cost: CostKind = CostKind.PRED_SUM, *, backend="det",
                          seed=0, bundle=None, trace=None):
    """Exact triangle count with the surrogate scheme (space_efficient.py:147-176).

    Returns (total, RunResult) whose per-rank `triangles`, `data_msgs_sent`,
    `data_msgs_to`, `bytes_sent` and `partition_bytes` match the reference.
    This single-device form evaluates every rank's work on one GPU; see
    distributed.count_space_surrogate_dist for one rank per GPU over NCCL.
    """
    ranges = partition_ranges(g, cost, nranks)
    bounds = range_bounds(ranges)
    dev = g.eff_indptr.device
    bd = torch.as_tensor(bounds).to(dev)
    t0 = time.perf_counter()
    if g.n >= 3:
        partials = count_middle(g, 0, g.n, bounds=bd).cpu().numpy()
    else:
        partials = np.zeros(nranks, dtype=np.int64)
    wall = time.perf_counter() - t0
    census, words = surrogate_census(g, bd, nranks)
    ip = g.eff_indptr.cpu().numpy()
    metrics = []
    for r in range(nranks):
        m = RankMetrics(rank=r, nranks=nranks)
        m.triangles = int(partials[r])
        m.data_msgs_to = census[r].astype(np.int64).copy()
        m.data_msgs_sent = int(census[r].sum())
        m.completion_msgs_sent = nranks - 1
        m.bytes_sent = WORD_BYTES * (int(words[r]) + (nranks - 1))
        m.partition_bytes = _partition_bytes(ip, int(bounds[r]), int(bounds[r + 1]))
        metrics.append(m)
    total = int(partials.sum())
    return total, RunResult(results=[total] + [None] * (nranks - 1), metrics=metrics, wall=wall)


def direct_census(g: Graph, bounds_dev, P):
    """(requests[P,P], reply_words[P]) of the direct scheme's per-pair
    messages (space_efficient.py:207-213, runtime.py:139-149)."""
    dev = g.eff_indptr.device
    req = torch.empty(P * P, dtype=torch.int64, device=dev)
    words = torch.empty(P, dtype=torch.int64, device=dev)
    _lib.call("tc_direct_census", _lib.ptr(g.eff_indptr), _lib.ptr(g.eff_indices), g.n, _lib.ptr(bounds_dev),
              int(P), _lib.ptr(req), _lib.ptr(words), _lib.stream())
    return req.view(P, P).cpu().numpy(), words.cpu().numpy()


def direct_metrics(r, P, partial, req, words, pbytes):
    """RankMetrics of rank r under the reference's direct-scheme accounting:
    one 2-word TASK_REQUEST per cross pair, one (2 + d^_u)-word DATA reply
    per request served, P-1 completion notifiers (space_efficient.py:188-231)."""
    m = RankMetrics(rank=r, nranks=P)
    m.triangles = int(partial)
    m.requests_to = np.asarray(req[r], np.int64).copy()
    m.requests_sent = int(m.requests_to.sum())
    m.data_msgs_to = np.asarray(req[:, r], np.int64).copy()
    m.data_msgs_sent = int(m.data_msgs_to.sum())
    m.completion_msgs_sent = P - 1
    m.bytes_sent = WORD_BYTES * (2 * m.requests_sent + int(words[r]) + (P - 1))
    m.partition_bytes = int(pbytes)
    return m


def count_space_direct(g: Graph, nranks: int, cost: CostKind = CostKind.PRED_SUM, *, backend="det", seed=0,
                       trace=None):
    """Exact triangle count with the direct request/response scheme
    (space_efficient.py:234-262).

    Returns (total, RunResult).  A rank's `triangles` is the lowest-vertex
    count of its range (the owner of v intersects N^_v with every fetched
    N^_u, space_efficient.py:206-219), its `requests_to` / `data_msgs_to` /
    `bytes_sent` follow the reference's one-request-per-cross-pair model.
    This single-device form evaluates every rank on one GPU; see
    distributed.count_space_direct_dist for one rank per GPU (deduplicated
    rank-level pull over NCCL)."""
    ranges = partition_ranges(g, cost, nranks)
    bounds = range_bounds(ranges)
    dev = g.eff_indptr.device
    bd = torch.as_tensor(bounds).to(dev)
    t0 = time.perf_counter()
    if g.n >= 3:
        partials = count_lowest(g, 0, g.n, bounds=bd).cpu().numpy()
    else:
        partials = np.zeros(nranks, dtype=np.int64)
    wall = time.perf_counter() - t0
    req, words = direct_census(g, bd, nranks)
    ip = g.eff_indptr.cpu().numpy()
    metrics = [direct_metrics(r, nranks, partials[r], req, words,
                              _partition_bytes(ip, int(bounds[r]), int(bounds[r + 1])))
               for r in range(nranks)]
    total = int(partials.sum())
    return total, RunResult(results=[total] + [None] * (nranks - 1), metrics=metrics, wall=wall)
