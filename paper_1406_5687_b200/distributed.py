"""One rank per GPU: the paper's space-efficient non-overlapping partition
with the surrogate exchange (space_efficient.py:81-176),
over torch.distributed (NCCL between B200s; gloo in the CPU tests).

Rank r owns the consecutive canonical range V_r = [b_r, b_{r+1}) balanced by
PRED_SUM (partitioning.py:139-141) and keeps ONLY the forward lists N^_v of
its own nodes (a "shard": local CSR + ids).  Protocol, bulk-synchronous:

  1. records   owner-change scan of the shard: one (v, dest) per remote rank
               dest > r touched by N^_v (LastProc dedup, _kernels.py:94-126);
               upper-triangular -- ranks only ever send to higher ranks.
  2. sizes     all_to_all of per-destination (#lists, #ids): replaces the
               reference's COMPLETION notifiers (space_efficient.py:132-139).
  3. exchange  all_to_all_single of the packed lists (node ids + lengths)
               and of the concatenated N^_v ids (NCCL send/recv pairs).
  4. count     the middle-vertex engine over owned u: table N^_u from the
               shard, segments = suffixes after u of local lists and of the
               received lists -- exactly surrogate_count_list's work
               (_kernels.py:70-80) -- so the rank's partial is the reference's
               per-rank `triangles` (middle-vertex attribution).
  5. reduce    all_reduce(SUM) of the uint64 partials (reduce_sum,
               runtime.py:255-259, 402-414).

The per-rank device work goes through `ops` (DeviceOps: libtcb200 kernels);
the CPU tests inject a numpy implementation of the same five primitives to
check the protocol with gloo at world_size 2.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .results import WORD_BYTES, RankMetrics


@dataclass
class Shard:
    """The forward lists of one rank's node range [lo, hi)."""

    lo: int
    hi: int
    indptr: torch.Tensor   # int64[hi - lo + 1], local offsets (indptr[0] == 0)
    indices: torch.Tensor  # int32[m_local (+4 padding)], global canonical ids

    @property
    def m(self):
        return int(self.indptr[-1])


def shard_of(g, lo, hi, device=None) -> Shard:
    """Cut rank [lo, hi)'s forward lists out of a (replicated) Graph."""
    e0, e1 = int(g.eff_indptr[lo]), int(g.eff_indptr[hi])
    dev = device or g.eff_indptr.device
    ip = (g.eff_indptr[lo: hi + 1] - e0).to(dev).contiguous()
    ix = torch.zeros(e1 - e0 + 4, dtype=torch.int32, device=dev)
    ix[: e1 - e0] = g.eff_indices[e0:e1].to(dev)
    return Shard(lo, hi, ip, ix[: e1 - e0])


class DeviceOps:
    """The rank-local primitives on the B200 (libtcb200 C ABI)."""

    def __init__(self):
        from . import _lib

        self._lib = _lib

    def records(self, shard: Shard, bounds, P, rank):
        """(rec_v int32 global ids grouped by dest, counts[P]) of step 1."""
        L = self._lib
        dev = shard.indptr.device
        nloc = shard.hi - shard.lo
        # the shard's CSR is indexed locally: shift bounds by lo and ids stay global
        b = torch.as_tensor(np.asarray(bounds, np.int64)).to(dev)
        cap = max(1, nloc * (P - 1))
        rec_v = torch.empty(cap, dtype=torch.int32, device=dev)
        rec_d = torch.empty(cap, dtype=torch.int32, device=dev)
        counts = torch.empty(P, dtype=torch.int64, device=dev)
        nrec = ctypes.c_int64()
        L.call("tc_surrogate_records", L.ptr(shard.indptr), L.ptr(shard.indices), nloc, L.ptr(b), P, rank, shard.lo,
               L.ptr(rec_v), L.ptr(rec_d), cap, L.ptr(counts), ctypes.byref(nrec), L.stream())
        k = nrec.value
        return rec_v[:k], counts.cpu().numpy()

    def pack(self, shard: Shard, rec_v):
        """(lengths int64[k], ids int32[...]) of the N^_v lists of records."""
        L = self._lib
        dev = shard.indptr.device
        k = int(rec_v.numel())
        loc = (rec_v - shard.lo).to(torch.int32).contiguous()
        offs = torch.empty(k + 1, dtype=torch.int64, device=dev)
        tot = ctypes.c_int64()
        L.call("tc_surrogate_pack_sizes", L.ptr(shard.indptr), L.ptr(loc), k, L.ptr(offs), ctypes.byref(tot), L.stream())
        ids = torch.empty(max(tot.value, 1), dtype=torch.int32, device=dev)
        L.call("tc_surrogate_pack", L.ptr(shard.indptr), L.ptr(shard.indices), L.ptr(loc), k, L.ptr(offs), L.ptr(ids),
               L.stream())
        return offs[1:] - offs[:-1], ids[: tot.value]

    def count(self, shard: Shard, recv_len, recv_ids, bounds=None):
        """Triangles with middle vertex in the shard's range (step 4)."""
        from .space_efficient import count_segments, owner_segments

        L = self._lib
        dev = shard.indptr.device
        nloc = shard.hi - shard.lo
        if nloc == 0:
            return 0
        # pool = local ids ++ received ids (16-byte aligned, padded)
        ml, mr = shard.m, int(recv_ids.numel())
        base_r = (ml + 3) // 4 * 4
        pool = torch.zeros(base_r + mr + 4, dtype=torch.int32, device=dev)
        pool[:ml] = shard.indices[:ml]
        pool[base_r: base_r + mr] = recv_ids
        owners, segs = [], []
        o1, s1, k1 = owner_segments(shard.indptr, pool[:ml] if ml else pool[:1], shard.lo, shard.hi, 0)
        if k1:
            owners.append(o1[:k1])
            segs.append(s1[: 2 * k1])
        if recv_len.numel():
            roffs = torch.zeros(recv_len.numel() + 1, dtype=torch.int64, device=dev)
            roffs[1:] = torch.cumsum(recv_len.to(dev), 0)
            o2, s2, k2 = owner_segments(roffs, recv_ids if mr else pool[:1], shard.lo, shard.hi, base_r)
            if k2:
                owners.append(o2[:k2])
                segs.append(s2[: 2 * k2])
        if not owners:
            return 0
        owner = torch.cat(owners).contiguous()
        seg = torch.cat(segs).contiguous()
        return int(count_segments(shard.indptr, shard.indices, pool, owner, seg, int(owner.numel()), nloc))


def _a2a_counts(counts_np, group, device):
    """all_to_all of one int64 per peer (step 2)."""
    P = len(counts_np)
    send = torch.as_tensor(np.asarray(counts_np, np.int64)).to(device)
    recv = torch.empty(P, dtype=torch.int64, device=device)
    dist.all_to_all_single(recv, send, group=group)
    return recv.cpu().numpy()


def surrogate_rank(shard: Shard, bounds, group=None, ops=None, device=None):
    """Run steps 1-5 on this rank; returns (total, RankMetrics)."""
    ops = ops or DeviceOps()
    P = dist.get_world_size(group)
    rank = dist.get_rank(group)
    device = device or shard.indptr.device
    met = RankMetrics(rank=rank, nranks=P)
    met.partition_bytes = WORD_BYTES * ((shard.hi - shard.lo) + 1 + shard.m)

    rec_v, counts = ops.records(shard, bounds, P, rank)                # 1
    lens, ids = ops.pack(shard, rec_v)
    lens_np = np.asarray(lens.cpu() if isinstance(lens, torch.Tensor) else lens, np.int64)
    # per-destination list counts and id counts (records are grouped by dest)
    id_counts = np.zeros(P, np.int64)
    start = 0
    for j in range(P):
        id_counts[j] = int(lens_np[start: start + counts[j]].sum())
        start += int(counts[j])
    met.data_msgs_to = counts.astype(np.int64).copy()
    met.data_msgs_sent = int(counts.sum())
    met.completion_msgs_sent = P - 1
    met.bytes_sent = WORD_BYTES * (2 * int(counts.sum()) + int(id_counts.sum()) + (P - 1))

    rcounts = _a2a_counts(counts, group, device)                      # 2
    rids = _a2a_counts(id_counts, group, device)
    recv_len = torch.empty(int(rcounts.sum()), dtype=torch.int64, device=device)
    dist.all_to_all_single(recv_len, torch.as_tensor(lens_np).to(device),        # 3
                           output_split_sizes=rcounts.tolist(), input_split_sizes=counts.tolist(), group=group)
    recv_ids = torch.empty(int(rids.sum()), dtype=torch.int32, device=device)
    send_ids = ids if isinstance(ids, torch.Tensor) else torch.as_tensor(ids)
    dist.all_to_all_single(recv_ids, send_ids.to(device).to(torch.int32),
                           output_split_sizes=rids.tolist(), input_split_sizes=id_counts.tolist(), group=group)

    part = ops.count(shard, recv_len, recv_ids)                       # 4
    met.triangles = int(part)
    t = torch.tensor([int(part)], dtype=torch.int64, device=device)
    dist.all_reduce(t, group=group)                                   # 5
    return int(t.item()), met


def count_space_surrogate_dist(g, cost=None, group=None, ops=None):
    """Multi-GPU count_space_surrogate: every rank holds the (replicated,
    identically built) graph g, keeps only its shard for the count, and
    returns (total, this rank's RankMetrics)."""
    from .partitioning import CostKind, partition_ranges, range_bounds

    cost = cost or CostKind.PRED_SUM
    P = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bounds = range_bounds(partition_ranges(g, cost, P))
    shard = shard_of(g, int(bounds[rank]), int(bounds[rank + 1]))
    return surrogate_rank(shard, bounds, group=group, ops=ops)


def emulate_ranks(g, P, cost=None, ops=None):
    """Runs the same five steps for all P ranks in one process, passing the
    packed buffers between ranks directly instead of through collectives.
    Used to check the per-rank device kernels of the multi-GPU path on one
    GPU (no rank ever waits on another, so nothing spins).  Returns
    (total, [RankMetrics])."""
    from .partitioning import CostKind, partition_ranges, range_bounds

    cost = cost or CostKind.PRED_SUM
    ops = ops or DeviceOps()
    bounds = range_bounds(partition_ranges(g, cost, P))
    shards = [shard_of(g, int(bounds[r]), int(bounds[r + 1])) for r in range(P)]
    mets = [RankMetrics(rank=r, nranks=P) for r in range(P)]
    outbox = {}  # (src, dst) -> (lens, ids)
    for r, sh in enumerate(shards):
        rec_v, counts = ops.records(sh, bounds, P, r)
        lens, ids = ops.pack(sh, rec_v)
        lens_np = np.asarray(lens.cpu() if isinstance(lens, torch.Tensor) else lens, np.int64)
        ids_t = ids if isinstance(ids, torch.Tensor) else torch.as_tensor(ids)
        start = istart = 0
        for j in range(P):
            c = int(counts[j])
            nid = int(lens_np[start: start + c].sum())
            if c:
                outbox[(r, j)] = (lens_np[start: start + c], ids_t[istart: istart + nid])
            start += c
            istart += nid
        m = mets[r]
        m.partition_bytes = WORD_BYTES * ((sh.hi - sh.lo) + 1 + sh.m)
        m.data_msgs_to = counts.astype(np.int64).copy()
        m.data_msgs_sent = int(counts.sum())
        m.completion_msgs_sent = P - 1
        m.bytes_sent = WORD_BYTES * (2 * int(counts.sum()) + int(istart) + (P - 1))
    total = 0
    for r, sh in enumerate(shards):
        dev = sh.indptr.device
        parts = [outbox[(s, r)] for s in range(P) if (s, r) in outbox]
        recv_len = torch.as_tensor(np.concatenate([p[0] for p in parts]) if parts else np.zeros(0, np.int64)).to(dev)
        recv_ids = torch.cat([p[1].to(dev) for p in parts]) if parts else torch.zeros(0, dtype=torch.int32, device=dev)
        mets[r].triangles = int(ops.count(sh, recv_len, recv_ids))
        total += mets[r].triangles
    return total, mets
