"""Dynamic load balancing (mirrors dynamic_lb.py:1-209 of the reference).

The paper's coordinator/worker scheme becomes, on the
B200, a device task queue: plan_tasks() is computed on the GPU with the
reference's exact rule (half the cost split evenly into the workers' initial
tasks, Eq. 1; then tasks of ceil(remaining/(P-1)) cost, Eq. 2), and
count_dynamic() executes every task in ONE launch of the lowest-vertex
engine whose warps pull cost-balanced chunks from a global atomic counter,
writing one exact partial per task.  Per-worker metrics are produced by a
deterministic emulation of the coordinator's FIFO service (each queued task
goes to the least-loaded worker), so RunResult keeps the reference's meaning.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .graph import Graph
from .partitioning import CostKind, NodeRange, balanced_ranges, node_costs, _dev_costs
from .results import RankMetrics, RunResult
from .sequential import count_lowest


@dataclass(frozen=True)
class Task:
    """Counting work for t consecutive nodes starting at v; atomic at t=1."""

    v: int
    t: int

    def __post_init__(self):
        if self.t < 1 or self.v < 0:
            raise ValueError(f"bad task ({self.v}, {self.t})")


@dataclass(frozen=True)
class TaskPlan:
    """Initial half-assignment plus the coordinator's queue (dynamic_lb.py:46-61)."""

    split: int
    initial: list
    queue: list
    targets: np.ndarray
    total_cost: int


def task_cost(costs, task: Task) -> int:
    if isinstance(costs, torch.Tensor):
        return int(costs[task.v: task.v + task.t].sum())
    return int(np.asarray(costs)[task.v: task.v + task.t].sum())


def plan_tasks(costs, nranks: int) -> TaskPlan:
    """Deterministic task plan for P-1 workers (dynamic_lb.py:68-109), on the device."""
    if nranks < 2:
        raise ValueError("dynamic scheme needs a coordinator plus at least one worker")
    c = _dev_costs(costs)
    n = int(c.numel())
    dev = c.device
    cc = c if n else torch.zeros(1, dtype=torch.int64, device=dev)
    ib = torch.empty(nranks, dtype=torch.int64, device=dev)
    qv = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    qt = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    tg = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    split, nq, total = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _lib.call("tc_plan_tasks", _lib.ptr(cc), n, int(nranks), _lib.ptr(ib), _lib.ptr(qv), _lib.ptr(qt),
              _lib.ptr(tg), ctypes.byref(split), ctypes.byref(nq), ctypes.byref(total), _lib.stream())
    q = nq.value
    b = ib.cpu().numpy()
    initial = [NodeRange(int(b[i]), int(b[i + 1] - b[i])) for i in range(nranks - 1)]
    qv_h, qt_h = qv[:q].cpu().numpy(), qt[:q].cpu().numpy()
    queue = [Task(int(v), int(t)) for v, t in zip(qv_h, qt_h)]
    return TaskPlan(split=int(split.value), initial=initial, queue=queue,
                    targets=tg[:q].cpu().numpy().astype(np.float64), total_cost=int(total.value))


def count_task(g: Graph, task: Task) -> int:
    """Triangles charged to the task's node range (lowest-vertex attribution)."""
    if task.v + task.t > g.n:
        raise ValueError(f"task ({task.v}, {task.t}) exceeds node count {g.n}")
    return int(count_lowest(g, task.v, task.v + task.t).item())


def count_dynamic(g: Graph, nranks: int, cost: CostKind = CostKind.DEGREE, *, backend="det", seed=0,
                  static_only=False, trace=None):
    """Exact triangle count under dynamic load balancing (dynamic_lb.py:176-209).

    Returns (total, RunResult).  `backend`, `seed` and `trace` address the
    reference's simulated runtime and are accepted for API compatibility; on
    the B200 the queue is a device atomic counter.
    """
    if nranks < 2:
        raise ValueError("count_dynamic needs at least 2 ranks (coordinator + worker)")
    costs = node_costs(g, cost)
    if static_only:
        initial = balanced_ranges(costs, NodeRange(0, g.n), nranks - 1)
        queue = []
    else:
        plan = plan_tasks(costs, nranks)
        initial, queue = plan.initial, plan.queue
    starts = [r.start for r in initial] + [t.v for t in queue]
    bounds = torch.as_tensor(np.asarray(starts + [g.n], dtype=np.int64)).to(g.eff_indptr.device)
    t0 = time.perf_counter()
    per_task = count_lowest(g, 0, g.n, bounds=bounds).cpu().numpy() if g.n else np.zeros(len(starts), np.int64)
    wall = time.perf_counter() - t0
    cost_h = costs.cpu().numpy() if g.n else np.zeros(0, np.int64)
    pref = np.concatenate([[0], np.cumsum(cost_h)])

    metrics = [RankMetrics(rank=r, nranks=nranks) for r in range(nranks)]
    load = np.zeros(nranks, dtype=np.int64)
    for w, r in enumerate(initial, start=1):
        if r.count:
            m = metrics[w]
            m.triangles += int(per_task[w - 1])
            m.tasks_executed += 1
            m.task_log.append((r.start, r.count))
            load[w] += pref[r.stop] - pref[r.start]
    for i, t in enumerate(queue):
        w = 1 + int(np.argmin(load[1:]))
        m = metrics[w]
        m.triangles += int(per_task[len(initial) + i])
        m.tasks_executed += 1
        m.requests_sent += 1
        m.requests_to[0] += 1
        m.task_log.append((t.v, t.t))
        load[w] += pref[t.v + t.t] - pref[t.v]
    for m in metrics[1:]:  # the final request answered with TERMINATE
        m.requests_sent += 1
        m.requests_to[0] += 1
        m.bytes_sent = 2 * 8 * m.requests_sent  # request_msg words=2 (runtime.py:93-94)
    metrics[0].bytes_sent = 8 * (3 * len(queue) + (nranks - 1))  # assign 3 words, terminate 1
    total = int(sum(m.triangles for m in metrics))
    return total, RunResult(results=[total] + [None] * (nranks - 1), metrics=metrics, wall=wall)
