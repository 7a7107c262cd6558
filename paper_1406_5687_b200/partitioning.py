"""Per-node costs and balanced consecutive node ranges (mirrors
partitioning.py:1-189).  Costs and prefix searches run on the device; the
small boundary arrays come back to the host like the reference's."""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .graph import Graph
from .results import WORD_BYTES


class CostKind(enum.Enum):
    """Per-node work estimates f(v) (partitioning.py:22-45)."""

    UNIT = "unit"
    DEGREE = "degree"
    SUCC_SUM = "succsum"
    PRED_SUM = "predsum"

    @classmethod
    def parse(cls, name):
        try:
            return cls(name.lower())
        except ValueError:
            raise ValueError(
                f"unknown cost function {name!r}; pick from {[k.value for k in cls]}"
            ) from None


_KIND_CODE = {CostKind.UNIT: 0, CostKind.DEGREE: 1, CostKind.SUCC_SUM: 2, CostKind.PRED_SUM: 3}


@dataclass(frozen=True)
class NodeRange:
    """A consecutive run of canonical node ids: [start, start + count)."""

    start: int
    count: int

    def __post_init__(self):
        if self.start < 0 or self.count < 0:
            raise ValueError(f"bad node range ({self.start}, {self.count})")

    @property
    def stop(self):
        return self.start + self.count


@dataclass(frozen=True)
class Partition:
    """One rank's share: the forward lists of its core node range."""

    rank: int
    core: NodeRange
    edge_count: int
    boundary: np.ndarray

    @property
    def node_count(self):
        return self.core.count + len(self.boundary)


def node_costs(g: Graph, kind: CostKind) -> torch.Tensor:
    """f(v) over all canonical nodes as a device int64 tensor (partitioning.py:79-92)."""
    if kind not in _KIND_CODE:
        raise ValueError(f"unknown cost kind {kind!r}")
    out = torch.empty(max(g.n, 1), dtype=torch.int64, device=g.eff_indptr.device)
    _lib.call("tc_node_costs", _KIND_CODE[kind], _lib.ptr(g.eff_indptr), _lib.ptr(g.eff_indices),
              _lib.ptr(g.deg), _lib.ptr(g.eff_deg), g.n, _lib.ptr(out), _lib.stream())
    return out[: g.n]


def _dev_costs(costs):
    dev = _lib.device()
    if isinstance(costs, torch.Tensor):
        return costs.to(dev, torch.int64).contiguous()
    return torch.as_tensor(np.asarray(costs, dtype=np.int64)).to(dev)


def balanced_bounds(costs, start, count, k) -> torch.Tensor:
    """Device int64[k+1] boundaries of balanced_ranges (partitioning.py:95-122)."""
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    c = _dev_costs(costs)
    b = torch.empty(k + 1, dtype=torch.int64, device=c.device)
    cp = c if c.numel() else torch.zeros(1, dtype=torch.int64, device=c.device)
    _lib.call("tc_balanced_bounds", _lib.ptr(cp), int(start), int(count), int(k), _lib.ptr(b),
              _lib.stream())
    return b


def balanced_ranges(costs, span: NodeRange, k: int) -> list:
    """Split `span` into k consecutive ranges of roughly equal total cost
    (partitioning.py:95-122): cut j after the smallest index whose inclusive
    prefix reaches ceil(j*total/k); all-zero totals split nodes equally."""
    b = balanced_bounds(costs, span.start, span.count, k).cpu().numpy()
    return [NodeRange(int(b[i]), int(b[i + 1] - b[i])) for i in range(k)]


def range_bounds(ranges) -> np.ndarray:
    """Boundary array b of length k+1 with range i = [b[i], b[i+1])."""
    bounds = np.empty(len(ranges) + 1, dtype=np.int64)
    for i, r in enumerate(ranges):
        bounds[i] = r.start
    bounds[-1] = ranges[-1].stop
    return bounds


def owner_of(bounds, v) -> int:
    """Rank owning node v under the given boundary array."""
    return int(np.searchsorted(np.asarray(bounds), v, side="right")) - 1


def partition_ranges(g: Graph, kind: CostKind, k: int) -> list:
    """Balanced core ranges over the whole node set."""
    return balanced_ranges(node_costs(g, kind), NodeRange(0, g.n), k)


def build_partition(g: Graph, core: NodeRange, rank: int) -> Partition:
    if core.stop > g.n:
        raise ValueError(f"core {core} exceeds node count {g.n}")
    lo, hi = int(g.eff_indptr[core.start]), int(g.eff_indptr[core.stop])
    owned = g.eff_indices[lo:hi]
    outside = torch.unique(owned)
    outside = outside[(outside < core.start) | (outside >= core.stop)]
    return Partition(rank=rank, core=core, edge_count=hi - lo,
                     boundary=outside.cpu().numpy().astype(np.int64))


def partition_bytes_nonoverlapping(p: Partition) -> int:
    """CSR words of a non-overlapping partition (partitioning.py:155-158)."""
    return WORD_BYTES * (p.core.count + 1 + p.edge_count)


def partition_bytes_overlapping_estimate(g: Graph, core: NodeRange) -> int:
    """Closure-based partition size (partitioning.py:161-179)."""
    fip, fix = g.full_indptr, g.full_indices
    lo, hi = int(fip[core.start]), int(fip[core.stop])
    dev = fix.device
    closure = torch.unique(torch.cat([torch.arange(core.start, core.stop, dtype=torch.int32, device=dev),
                                      fix[lo:hi]]))
    return WORD_BYTES * (int(closure.numel()) + 1 + int(g.deg[closure.long()].sum()))


def graph_bytes_full(g: Graph) -> int:
    return WORD_BYTES * (g.n + 1 + 2 * g.m)


def graph_bytes_forward(g: Graph) -> int:
    return WORD_BYTES * (g.n + 1 + g.m)
