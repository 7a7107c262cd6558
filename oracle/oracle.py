"""CPU oracle for the triangle-counting hot path -- TEST INFRASTRUCTURE ONLY.

ctypes/numpy front end over ``oracle.c`` (a C restatement of the reference
``tricount`` package, /root/reference/pkg/src/tricount).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm may
import this module; the product package never does.

Parity of this oracle is pinned by tests/test_oracle_golden.py against vectors
produced by running the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_P64 = ctypes.POINTER(ctypes.c_int64)


def _ptr(a):
    return a.ctypes.data_as(_P64)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        src = os.path.join(_HERE, "oracle.c")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        L = ctypes.CDLL(path)
        i64, p = ctypes.c_int64, _P64
        L.or_normalize.argtypes = [p, i64, p, p, p]
        L.or_build_graph.argtypes = [i64, p, i64, p, p, p, p, p, p, p, p, p]
        L.or_intersect_size.argtypes = [p, i64, p, i64]
        L.or_intersect_size.restype = i64
        L.or_count_node_range.argtypes = [p, p, i64, i64]
        L.or_count_node_range.restype = i64
        L.or_node_costs.argtypes = [ctypes.c_int, i64, p, p, p, p]
        L.or_balanced_bounds.argtypes = [p, i64, i64, i64, p]
        L.or_plan_tasks.argtypes = [p, i64, i64, p, p, p, p,
                                    ctypes.POINTER(ctypes.c_double), p, p]
        L.or_surrogate.argtypes = [p, p, i64, p, i64, p, p]
        L.or_direct.argtypes = [p, p, i64, p, i64, p, p, p]
        L.or_surrogate_count_list.argtypes = [p, p, i64, i64, p, i64]
        L.or_surrogate_count_list.restype = i64
        L.or_pa_num_edges.argtypes = [i64, i64]
        L.or_pa_num_edges.restype = i64
        L.or_pa_edge_list.argtypes = [i64, i64, ctypes.c_uint64, p, p]
        L.or_count_tasks_threaded.argtypes = [p, p, p, p, i64, ctypes.c_int]
        L.or_count_tasks_threaded.restype = i64
        _LIB = L
    return _LIB


def _i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


# -- graph.py -----------------------------------------------------------------


def normalize(edges):
    """graph.py:76-103 -> (n, (m,2) int64 edges)."""
    e = _i64(edges).reshape(-1, 2)
    out = np.empty((max(len(e), 1), 2), dtype=np.int64)
    m = np.zeros(1, np.int64)
    n = np.zeros(1, np.int64)
    rc = lib().or_normalize(_ptr(e), len(e), _ptr(out), _ptr(m), _ptr(n))
    if rc == -1:
        raise ValueError("negative node id in edge list")
    return int(n[0]), out[: int(m[0])].copy()


@dataclass
class OGraph:
    n: int
    m: int
    eff_indptr: np.ndarray
    eff_indices: np.ndarray
    full_indptr: np.ndarray
    full_indices: np.ndarray
    relabel: np.ndarray
    orig_ids: np.ndarray
    deg: np.ndarray
    eff_deg: np.ndarray


def build_graph(n, edges, order=None, full=True):
    """graph.py:106-153 (order=None: degree order; else _build_graph_input_order)."""
    e = _i64(edges).reshape(-1, 2)
    m = len(e)
    arr = lambda k: np.zeros(max(k, 1), dtype=np.int64)  # noqa: E731
    eff_indptr, eff_indices = arr(n + 1), arr(m)
    full_indptr, full_indices = arr(n + 1), arr(2 * m)
    relabel, orig_ids, deg, eff_deg = arr(n), arr(n), arr(n), arr(n)
    o = _i64(order) if order is not None else None
    rc = lib().or_build_graph(
        n, _ptr(e), m, _ptr(o) if o is not None else None,
        _ptr(eff_indptr), _ptr(eff_indices),
        _ptr(full_indptr) if full else None, _ptr(full_indices) if full else None,
        _ptr(relabel), _ptr(orig_ids), _ptr(deg), _ptr(eff_deg))
    if rc != 0:
        raise ValueError("edge id out of range")
    return OGraph(n, m, eff_indptr[: n + 1], eff_indices[:m], full_indptr[: n + 1],
                  full_indices[: 2 * m], relabel[:n], orig_ids[:n], deg[:n], eff_deg[:n])


# -- _kernels.py / sequential.py ----------------------------------------------


def intersect_size(a, b):
    a, b = _i64(a), _i64(b)
    return int(lib().or_intersect_size(_ptr(a), len(a), _ptr(b), len(b)))


def count_node_range(indptr, indices, start, stop):
    """_kernels.py:40-52."""
    ip, ix = _i64(indptr), _i64(indices)
    return int(lib().or_count_node_range(_ptr(ip), _ptr(ix), int(start), int(stop)))


def count_triangles(g: OGraph):
    """sequential.py:30-34."""
    if g.n < 3:
        return 0
    return count_node_range(g.eff_indptr, g.eff_indices, 0, g.n)


def count_triangles_brute(n, full_indptr, full_indices):
    """Independent dense oracle (sequential.py:37-51), small n only."""
    if n < 3:
        return 0
    adj = np.zeros((n, n), dtype=bool)
    for v in range(n):
        adj[v, full_indices[full_indptr[v]: full_indptr[v + 1]]] = True
    a = adj.astype(np.int64)
    return int(np.trace(a @ a @ a) // 6)


# -- partitioning.py / dynamic_lb.py / space_efficient.py ---------------------

COST_KINDS = {"unit": 0, "degree": 1, "succsum": 2, "predsum": 3}


def node_costs(g: OGraph, kind: str):
    """partitioning.py:79-92."""
    out = np.zeros(max(g.n, 1), np.int64)
    ip, ix, dg = _i64(g.eff_indptr), _i64(g.eff_indices), _i64(g.deg)
    lib().or_node_costs(COST_KINDS[kind], g.n, _ptr(ip), _ptr(ix), _ptr(dg), _ptr(out))
    return out[: g.n]


def balanced_bounds(costs, start, count, k):
    """partitioning.py:95-122 -> bounds[k+1]."""
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    c = _i64(costs) if len(costs) else np.zeros(1, np.int64)
    b = np.zeros(k + 1, np.int64)
    lib().or_balanced_bounds(_ptr(c), int(start), int(count), int(k), _ptr(b))
    return b


def plan_tasks(costs, nranks):
    """dynamic_lb.py:68-109 -> dict(split, initial_bounds, queue [(v,t)], targets, total)."""
    c = _i64(costs)
    n = len(c)
    cc = c if n else np.zeros(1, np.int64)
    ib = np.zeros(max(nranks, 2), np.int64)
    qv = np.zeros(max(n, 1), np.int64)
    qt = np.zeros(max(n, 1), np.int64)
    tg = np.zeros(max(n, 1), np.float64)
    split, nq, total = np.zeros(1, np.int64), np.zeros(1, np.int64), np.zeros(1, np.int64)
    rc = lib().or_plan_tasks(_ptr(cc), n, int(nranks), _ptr(split), _ptr(ib), _ptr(qv), _ptr(qt),
                             tg.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _ptr(nq),
                             _ptr(total))
    if rc == -1:
        raise ValueError("dynamic scheme needs a coordinator plus at least one worker")
    if rc == -2:
        raise ValueError("costs must be non-negative")
    q = int(nq[0])
    return dict(split=int(split[0]), initial_bounds=ib[:nranks].copy(),
                queue=list(zip(qv[:q].tolist(), qt[:q].tolist())), targets=tg[:q].copy(),
                total=int(total[0]))


def surrogate(g: OGraph, bounds):
    """Per-rank partials + LastProc census of count_space_surrogate
    (space_efficient.py:81-144)."""
    P = len(bounds) - 1
    b = _i64(bounds)
    partials = np.zeros(P, np.int64)
    census = np.zeros(P * P, np.int64)
    lib().or_surrogate(_ptr(_i64(g.eff_indptr)), _ptr(_i64(g.eff_indices)), g.n, _ptr(b), P,
                       _ptr(partials), _ptr(census))
    return partials, census.reshape(P, P)


def direct(g: OGraph, bounds):
    """Per-rank partials (lowest vertex), per-pair request matrix and reply
    words of count_space_direct (space_efficient.py:188-231)."""
    P = len(bounds) - 1
    b = _i64(bounds)
    partials = np.zeros(P, np.int64)
    req = np.zeros(P * P, np.int64)
    words = np.zeros(P, np.int64)
    lib().or_direct(_ptr(_i64(g.eff_indptr)), _ptr(_i64(g.eff_indices)), g.n, _ptr(b), P, _ptr(partials),
                    _ptr(req), _ptr(words))
    return partials, req.reshape(P, P), words


def surrogate_count_list(g: OGraph, lo, hi, x):
    """_kernels.py:70-80."""
    x = _i64(x) if len(x) else np.zeros(1, np.int64)
    nx = len(x) if len(x) and x.size else 0
    return int(lib().or_surrogate_count_list(_ptr(_i64(g.eff_indptr)), _ptr(_i64(g.eff_indices)),
                                             int(lo), int(hi), _ptr(x), nx))


def pa_edge_list(n, d, seed):
    """graph_io.py:102-112 / _kernels.py:129-178 -> (m,2) int64."""
    k = d // 2
    m = int(lib().or_pa_num_edges(n, k))
    src = np.empty(m, np.int64)
    dst = np.empty(m, np.int64)
    lib().or_pa_edge_list(n, k, ctypes.c_uint64(seed), _ptr(src), _ptr(dst))
    return np.column_stack([src, dst])


def count_tasks_threaded(indptr, indices, tasks_v, tasks_t, nthreads):
    """count_dynamic's worker loop (dynamic_lb.py:141-173) on host threads."""
    ip, ix = _i64(indptr), _i64(indices)
    tv, tt = _i64(tasks_v), _i64(tasks_t)
    return int(lib().or_count_tasks_threaded(_ptr(ip), _ptr(ix), _ptr(tv), _ptr(tt), len(tv),
                                             int(nthreads)))
