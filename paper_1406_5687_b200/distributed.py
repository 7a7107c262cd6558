"""One rank per GPU: the paper's space-efficient non-overlapping partition
with the surrogate exchange (space_efficient.py:81-176)
and the direct scheme as a deduplicated pull (space_efficient.py:179-262;
`direct_rank` below), over torch.distributed (NCCL between B200s; gloo in
the CPU tests).

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
from dataclasses import dataclass, field

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
    # derived from the shard's own lists only, built on first use (the pull
    # index of count_direct: local segments grouped by owner)
    cache: dict = field(default_factory=dict, repr=False, compare=False)

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

    def _local_plan(self, shard: Shard):
        """Engine plan over the shard's own lists (owned u, local
        predecessors), built once per shard: the part of step 4 that does
        not depend on what was received."""
        from .space_efficient import owner_segments, segments_csr

        L = self._lib
        plan = shard.cache.get("surrogate_local")
        if plan is None:
            nloc, ml = shard.hi - shard.lo, shard.m
            pool = torch.zeros(ml + 4, dtype=torch.int32, device=shard.indptr.device)  # aligned + padded
            pool[:ml] = shard.indices[:ml]
            owner, segs, k = owner_segments(shard.indptr, pool[: max(ml, 1)], shard.lo, shard.hi, 0)
            row, rsegs, cost = segments_csr(owner[:k].contiguous(), segs[: 2 * k].contiguous(), k, nloc,
                                            shard.indptr)
            h = ctypes.c_void_p()
            L.call("tc_plan_middle", L.ptr(shard.indptr), L.ptr(pool), L.ptr(row), L.ptr(rsegs), L.ptr(cost),
                   L.ptr(pool), 0, nloc, 0, nloc, None, 1, ctypes.byref(h), L.stream())
            plan = shard.cache["surrogate_local"] = _PlanHandle(h, (pool, row, rsegs, cost))
        return plan

    def count(self, shard: Shard, recv_len, recv_ids, bounds=None):
        """Triangles with middle vertex in the shard's range (step 4): the
        cached local plan plus one engine run over the received lists."""
        from .space_efficient import count_segments, owner_segments

        L = self._lib
        dev = shard.indptr.device
        nloc = shard.hi - shard.lo
        if nloc == 0:
            return 0
        out = torch.empty(2, dtype=torch.int64, device=dev)
        out[1:].zero_()
        L.call("tc_plan_run", self._local_plan(shard).handle, L.ptr(out), L.stream())
        mr = int(recv_ids.numel())
        if recv_len.numel() and mr:
            pool = torch.zeros(mr + 4, dtype=torch.int32, device=dev)  # aligned + padded
            pool[:mr] = recv_ids
            roffs = torch.zeros(recv_len.numel() + 1, dtype=torch.int64, device=dev)
            roffs[1:] = torch.cumsum(recv_len.to(dev), 0)
            o2, s2, k2 = owner_segments(roffs, pool[:mr], shard.lo, shard.hi, 0)
            if k2:
                out[1] = count_segments(shard.indptr, shard.indices, pool, o2[:k2].contiguous(),
                                        s2[: 2 * k2].contiguous(), k2, nloc)
        return int(out.sum().item())

    def requests(self, shard: Shard, bounds, P, rank):
        """Direct scheme, step 1: (req_ids int32 ascending, req_mult int64,
        counts[P] distinct ids per owner, ref_counts[P] per-pair requests)."""
        L = self._lib
        dev = shard.indptr.device
        nloc = shard.hi - shard.lo
        b = torch.as_tensor(np.asarray(bounds, np.int64)).to(dev)
        cap = max(1, shard.m)
        ids = torch.empty(cap, dtype=torch.int32, device=dev)
        mult = torch.empty(cap, dtype=torch.int64, device=dev)
        counts = torch.empty(P, dtype=torch.int64, device=dev)
        ref = torch.empty(P, dtype=torch.int64, device=dev)
        k = ctypes.c_int64()
        L.call("tc_direct_requests", L.ptr(shard.indptr), L.ptr(shard.indices), nloc, shard.hi, L.ptr(b), P,
               L.ptr(ids), L.ptr(mult), cap, L.ptr(counts), L.ptr(ref), ctypes.byref(k), L.stream())
        return ids[: k.value], mult[: k.value], counts.cpu().numpy(), ref.cpu().numpy()

    def count_direct(self, shard: Shard, req_ids, fetched_len, fetched_ids):
        """Direct scheme, step 4: count_node_range(lo, hi) over the shard's
        lists and the fetched N^_u (lowest-vertex attribution), with the
        middle-vertex engine: tables N^_u from the lookup CSR (own rows +
        fetched rows), segments = suffixes of the shard's own lists only,
        grouped by owner once per shard (Shard.cache)."""
        from .space_efficient import owner_segments, segments_csr

        L = self._lib
        dev = shard.indptr.device
        nloc = shard.hi - shard.lo
        if nloc == 0 or shard.m == 0:
            return 0
        nreq = int(req_ids.numel())
        n_rows = max(shard.hi, int(req_ids[-1].item()) + 1 if nreq else 0)
        indptr = torch.empty(n_rows + 1, dtype=torch.int64, device=dev)
        flen = fetched_len.to(dev, torch.int64).contiguous()
        L.call("tc_direct_table", L.ptr(shard.indptr), nloc, shard.lo, L.ptr(req_ids) if nreq else None,
               L.ptr(flen) if nreq else None, nreq, n_rows, L.ptr(indptr), L.stream())
        ml, mr = shard.m, int(fetched_ids.numel())
        pool = torch.zeros(ml + mr + 4, dtype=torch.int32, device=dev)  # +4: 16-byte chunk reads
        pool[:ml] = shard.indices[:ml]
        pool[ml: ml + mr] = fetched_ids
        key = ("pull", n_rows)
        idx = shard.cache.get(key)
        if idx is None:
            owner, segs, k = owner_segments(shard.indptr, pool[:ml], 0, n_rows, 0)
            idx = segments_csr(owner[:k].contiguous(), segs[: 2 * k].contiguous(), k, n_rows, indptr)
            shard.cache.clear()
            shard.cache[key] = idx
        row, rsegs, cost = idx
        out = torch.empty(1, dtype=torch.int64, device=dev)
        L.call("tc_count_middle", L.ptr(indptr), L.ptr(pool), L.ptr(row), L.ptr(rsegs), L.ptr(cost), L.ptr(pool),
               0, n_rows, 0, n_rows, None, 1, L.ptr(out), L.stream())
        return int(out.item())

class _PlanHandle:
    """A tc_plan_t plus the device arrays it points into."""

    __slots__ = ("handle", "keep")

    def __init__(self, handle, keep):
        self.handle, self.keep = handle, keep

    def __del__(self):
        try:
            if self.handle:
                from . import _lib
                _lib.lib().tc_plan_free(self.handle)
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass


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
    if ops is None:
        # the sharded pipeline's count (sharded.py): sizes, lengths and
        # plans stay on the device / on the shard, bounded exchange rounds,
        # the local engine overlapping the exchange; same partials and census
        from . import sharded as S

        key = ("surrogate_shard", P, rank, str(cost))
        sh = g._cache.get(key)
        if sh is None:
            sh = g._cache[key] = S.shard_from_graph(g, bounds, rank)
        return S.count_sharded(sh, group=group)
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


def _split_sums(values_np, counts_np):
    """Per-peer sums of a peer-grouped array."""
    out = np.zeros(len(counts_np), np.int64)
    start = 0
    for j, c in enumerate(np.asarray(counts_np, np.int64).tolist()):
        out[j] = int(np.asarray(values_np[start: start + c], np.int64).sum())
        start += c
    return out


def direct_rank(shard: Shard, bounds, group=None, ops=None, device=None):
    """The direct scheme on this rank as a deduplicated rank-level pull
    (space_efficient.py:179-231); returns (total, RankMetrics).

      1. requests  distinct remote ids named by the shard's lists, ascending
                   (= grouped by owner), with their per-pair multiplicity
      2. ask       all_to_all of the id counts, then of the ids and
                   multiplicities (the reference sends one TASK_REQUEST per
                   cross pair; here one id per distinct u and rank)
      3. serve     pack the requested N^_w lists, all_to_all them back
      4. count     count_node_range(lo, hi) over own + fetched lists
      5. reduce    all_reduce(SUM)

    The metrics keep the reference's per-pair accounting (requests_to,
    data_msgs_to, bytes_sent); wire_bytes is what the collectives moved."""
    ops = ops or DeviceOps()
    P = dist.get_world_size(group)
    rank = dist.get_rank(group)
    device = device or shard.indptr.device
    met = RankMetrics(rank=rank, nranks=P)
    met.partition_bytes = WORD_BYTES * ((shard.hi - shard.lo) + 1 + shard.m)

    req_ids, req_mult, counts, ref_counts = ops.requests(shard, bounds, P, rank)          # 1
    met.requests_to = np.asarray(ref_counts, np.int64).copy()
    met.requests_sent = int(met.requests_to.sum())
    rcounts = _a2a_counts(counts, group, device)                                            # 2
    recv_ids = torch.empty(int(rcounts.sum()), dtype=torch.int32, device=device)
    dist.all_to_all_single(recv_ids, req_ids.to(device, torch.int32), output_split_sizes=rcounts.tolist(),
                           input_split_sizes=counts.tolist(), group=group)
    recv_mult = torch.empty(int(rcounts.sum()), dtype=torch.int64, device=device)
    dist.all_to_all_single(recv_mult, req_mult.to(device, torch.int64), output_split_sizes=rcounts.tolist(),
                           input_split_sizes=counts.tolist(), group=group)

    lens, ids = ops.pack(shard, recv_ids)                                                   # 3
    lens_np = np.asarray(lens.cpu() if isinstance(lens, torch.Tensor) else lens, np.int64)
    mult_np = recv_mult.cpu().numpy()
    met.data_msgs_to = _split_sums(mult_np, rcounts)
    met.data_msgs_sent = int(met.data_msgs_to.sum())
    met.completion_msgs_sent = P - 1
    reply_words = int((mult_np * (2 + lens_np)).sum()) if lens_np.size else 0
    met.bytes_sent = WORD_BYTES * (2 * met.requests_sent + reply_words + (P - 1))
    reply_id_counts = _split_sums(lens_np, rcounts)
    fetched_id_counts = _a2a_counts(reply_id_counts, group, device)
    fetched_len = torch.empty(int(counts.sum()), dtype=torch.int64, device=device)
    dist.all_to_all_single(fetched_len, torch.as_tensor(lens_np).to(device), output_split_sizes=counts.tolist(),
                           input_split_sizes=rcounts.tolist(), group=group)
    fetched_ids = torch.empty(int(fetched_id_counts.sum()), dtype=torch.int32, device=device)
    send_ids = ids if isinstance(ids, torch.Tensor) else torch.as_tensor(ids)
    dist.all_to_all_single(fetched_ids, send_ids.to(device, torch.int32),
                           output_split_sizes=fetched_id_counts.tolist(),
                           input_split_sizes=reply_id_counts.tolist(), group=group)
    met.wire_bytes = int(12 * counts.sum() + 8 * rcounts.sum() + 4 * reply_id_counts.sum() + 16 * P)

    part = ops.count_direct(shard, req_ids, fetched_len, fetched_ids)                       # 4
    met.triangles = int(part)
    t = torch.tensor([int(part)], dtype=torch.int64, device=device)
    dist.all_reduce(t, group=group)                                                         # 5
    return int(t.item()), met


def count_space_direct_dist(g, cost=None, group=None, ops=None):
    """Multi-GPU count_space_direct (one rank per GPU): returns (total, this
    rank's RankMetrics)."""
    from .partitioning import CostKind, partition_ranges, range_bounds

    cost = cost or CostKind.PRED_SUM
    P = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bounds = range_bounds(partition_ranges(g, cost, P))
    shard = shard_of(g, int(bounds[rank]), int(bounds[rank + 1]))
    return direct_rank(shard, bounds, group=group, ops=ops)


def emulate_direct_ranks(g, P, cost=None, ops=None):
    """direct_rank's steps for all P ranks in one process (buffers passed
    directly).  Returns (total, [RankMetrics])."""
    from .partitioning import CostKind, partition_ranges, range_bounds

    cost = cost or CostKind.PRED_SUM
    ops = ops or DeviceOps()
    bounds = range_bounds(partition_ranges(g, cost, P))
    shards = [shard_of(g, int(bounds[r]), int(bounds[r + 1])) for r in range(P)]
    mets = [RankMetrics(rank=r, nranks=P) for r in range(P)]
    asks = []
    for r, sh in enumerate(shards):
        req_ids, req_mult, counts, ref = ops.requests(sh, bounds, P, r)
        asks.append((req_ids, req_mult, np.asarray(counts, np.int64)))
        mets[r].requests_to = np.asarray(ref, np.int64).copy()
        mets[r].requests_sent = int(mets[r].requests_to.sum())
        mets[r].partition_bytes = WORD_BYTES * ((sh.hi - sh.lo) + 1 + sh.m)
        mets[r].completion_msgs_sent = P - 1
    replies = {}  # (server, client) -> (lens, ids)
    for j, sh in enumerate(shards):
        words = 0
        to = np.zeros(P, np.int64)
        for i in range(P):
            ids_i, mult_i, counts_i = asks[i]
            a = int(counts_i[:j].sum())
            c = int(counts_i[j])
            if c == 0:
                continue
            lens, lists = ops.pack(sh, ids_i[a: a + c])
            lens_np = np.asarray(lens.cpu() if isinstance(lens, torch.Tensor) else lens, np.int64)
            mult_np = np.asarray(mult_i[a: a + c].cpu() if isinstance(mult_i, torch.Tensor) else mult_i[a: a + c],
                                 np.int64)
            to[i] = int(mult_np.sum())
            words += int((mult_np * (2 + lens_np)).sum())
            replies[(j, i)] = (lens_np, lists)
        mets[j].data_msgs_to = to
        mets[j].data_msgs_sent = int(to.sum())
        mets[j].bytes_sent = WORD_BYTES * (2 * mets[j].requests_sent + words + (P - 1))
    total = 0
    for i, sh in enumerate(shards):
        dev = sh.indptr.device
        parts = [replies[(j, i)] for j in range(P) if (j, i) in replies]
        flen = torch.as_tensor(np.concatenate([p[0] for p in parts]) if parts else np.zeros(0, np.int64)).to(dev)
        fids = (torch.cat([torch.as_tensor(p[1]).to(dev, torch.int32) for p in parts]) if parts
                else torch.zeros(0, dtype=torch.int32, device=dev))
        mets[i].triangles = int(ops.count_direct(sh, asks[i][0], flen, fids))
        total += mets[i].triangles
    return total, mets
