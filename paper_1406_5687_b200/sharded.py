"""The sharded multi-GPU pipeline: the paper's space-efficient algorithm on
non-overlapping node-range partitions from the
raw edge list to the total, one rank per GPU.

No rank ever holds the whole graph.  Rank r starts from its slice of the raw
pairs, and
  build   1. labels      all_reduce of per-label presence (MAX) and first
                         raveled position (MIN): the dense check and the
                         first-seen compaction of graph.py:92-99, replicated
          2. dedup       canonical keys all_to_all'd by hash, sorted + unique
                         per rank (np.unique(axis=0), graph.py:100-102)
          3. order       degrees all_reduce'd; ascending (degree, id) order
                         (graph.py:152), replicated O(n)
          4. orient      (lo, hi) pairs; out-degrees all_reduce'd; PRED_SUM
                         costs all_reduce'd -> the reference's partition
                         (partitioning.py:139-141); optionally re-balanced by
                         the middle-vertex engine's own cost (cost="engine")
          5. shard       pairs all_to_all'd to the owner of lo; local CSR
                         (rows sorted) + the engine's row-padded pool
  count   6. local       middle-vertex engine over the shard's own lists,
                         launched first so it overlaps the exchange
          7. exchange    per destination j > r (LastProc, _kernels.py:94-126)
                         the suffix of N^_v at or above b_j (from its 16-byte
                         chunk of the padded pool), padded, in
                         bounded rounds (a round = a group of consecutive
                         sender ranks); each round's lists are indexed and
                         counted on the device while the next round is in
                         flight
          8. reduce      all_reduce(SUM) of the uint64 partials
                         (reduce_sum, runtime.py:255-259)

Rank partials are the triangles whose middle vertex the rank owns: with the
PRED_SUM partition they equal the reference's count_space_surrogate
metrics[r].triangles, and the census / bytes_sent its data_msgs_to /
bytes_sent (space_efficient.py:116-144).

The per-rank steps are written once, as generators that yield their
collectives; `run_dist` executes them over torch.distributed (NCCL between
B200s, gloo in the CPU tests) and `emulate` runs P of them in lockstep in
one process (one GPU: the per-rank kernels run rank after rank, buffers are
passed directly, no rank ever waits on another) and reports each rank's
device time.  The device work goes through `ops` (ShardOps: libtcb200's
tc_shard_* kernels); the CPU tests inject a numpy implementation.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .results import WORD_BYTES, RankMetrics

POOL_HEAD = 512  # TC_POOL_HEAD (include/tcb200.h)
# Weight of an owner's table ids against its streamed probe ids in the
# engine-cost partition (cost="engine"): staging a table costs more per id
# than a probe (hashing + atomics), see DESIGN.md §4.
TAB_WEIGHT = int(__import__("os").environ.get("TCB_TAB_WEIGHT", "8"))
# Weight of a predecessor segment (one list suffix streamed for one owner)
# against one probe id.
SEG_WEIGHT = int(__import__("os").environ.get("TCB_SEG_WEIGHT", "2"))
# Weight of a node's own list (the owner packs and sends it to the ranks
# above) against one probe id.
SEND_WEIGHT = int(__import__("os").environ.get("TCB_SEND_WEIGHT", "16"))
INT32_MAX = 2**31 - 1


# ------------------------------------------------------------------ data

@dataclass
class ShardGraph:
    """One rank's part of the graph after the sharded build."""

    lo: int
    hi: int
    n: int                      # nodes of the whole graph
    m: int                      # edges of the whole graph
    bounds: np.ndarray          # int64[P+1], identical on every rank
    indptr: torch.Tensor        # int64[hi-lo+1], local offsets
    indices: torch.Tensor       # int32[m_local], canonical ids, rows ascending
    pool_indptr: torch.Tensor   # the engine's row-padded copy (rows at multiples of 4)
    pool: torch.Tensor          # view POOL_HEAD ids past its buffer's start
    relabel: torch.Tensor | None = None   # kept only with keep_maps=True (tests)
    orig_ids: torch.Tensor | None = None
    cache: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def m_local(self):
        return int(self.indices.numel())

    def resident_bytes(self):
        """Bytes of the rank's graph state (the partition: lists + offsets +
        the engine's padded copy)."""
        return sum(int(t.numel()) * t.element_size() for t in (self.indptr, self.indices, self.pool_indptr)) + \
            (int(self.pool.numel()) + POOL_HEAD) * 4


# ------------------------------------------------------------------ device ops

class ShardOps:
    """The per-rank device steps (libtcb200 tc_shard_* / tc_plan_*)."""

    def __init__(self, device=None):
        from . import _lib

        self.L = _lib
        self.dev = device or _lib.device()
        # timing = True brackets the rank's own device work (pack, receive
        # index, engine runs) with CUDA events on the streams it runs on;
        # busy_ms() is their sum -- the rank's cost for rebalance_gen, free of
        # the time spent waiting for peers
        self.timing = False
        self._busy = []

    def _tic(self, stream=None):
        if not self.timing:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream or torch.cuda.current_stream(self.dev))
        return e

    def _toc(self, e0, stream=None, label="engine"):
        if e0 is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(stream or torch.cuda.current_stream(self.dev))
            self._busy.append((e0, e1, label))

    def busy_ms(self, by_label=None):
        """Device time of the bracketed work since the last call (by_label:
        a dict that receives the split into pack / index / engine)."""
        torch.cuda.synchronize(self.dev)
        t = 0.0
        for a, b, label in self._busy:
            dt = a.elapsed_time(b)
            t += dt
            if by_label is not None:
                by_label[label] = by_label.get(label, 0.0) + dt
        self._busy = []
        return t

    # -- build --
    def minmax(self, pairs):
        lo, hi = ctypes.c_int32(), ctypes.c_int32()
        self.L.call("tc_shard_minmax", self.L.ptr(pairs), int(pairs.shape[0]), ctypes.byref(lo), ctypes.byref(hi),
                    self.L.stream())
        return lo.value, hi.value

    def label_scan(self, pairs, pos_base, K):
        present = torch.empty(max(K, 1), dtype=torch.uint8, device=self.dev)
        first = torch.empty(max(K, 1), dtype=torch.int32, device=self.dev)
        self.L.call("tc_shard_label_scan", self.L.ptr(pairs), int(pairs.shape[0]), int(pos_base), int(K),
                    self.L.ptr(present), self.L.ptr(first), self.L.stream())
        return present[:K], first[:K]

    def relabel_map(self, present, first, K):
        mp = torch.empty(max(K, 1), dtype=torch.int32, device=self.dev)
        n, dense = ctypes.c_int64(), ctypes.c_int32()
        self.L.call("tc_shard_relabel_map", self.L.ptr(present), self.L.ptr(first), int(K), self.L.ptr(mp),
                    ctypes.byref(n), ctypes.byref(dense), self.L.stream())
        return mp[:K], n.value, bool(dense.value)

    def keys(self, pairs, mp, P):
        m = int(pairs.shape[0])
        keys = torch.empty(max(m, 1), dtype=torch.int64, device=self.dev)
        counts = np.zeros(P, np.int64)
        self.L.call("tc_shard_keys", self.L.ptr(pairs), m, self.L.ptr(mp), int(P), self.L.ptr(keys),
                    counts.ctypes.data_as(ctypes.c_void_p), self.L.stream())
        return keys[: int(counts.sum())], counts

    def dedup(self, keys, n):
        k = int(keys.numel())
        out = torch.empty(max(k, 1), dtype=torch.int64, device=self.dev)
        kk = ctypes.c_int64()
        bits = max(1, int(n - 1).bit_length()) if n > 1 else 1
        self.L.call("tc_shard_dedup", self.L.ptr(keys), k, bits, self.L.ptr(out), ctypes.byref(kk), self.L.stream())
        return out[: kk.value]

    def degrees(self, ukeys, n):
        deg = torch.zeros(max(n, 1), dtype=torch.int32, device=self.dev)
        self.L.call("tc_shard_degrees", self.L.ptr(ukeys), int(ukeys.numel()), self.L.ptr(deg), self.L.stream())
        return deg[:n]

    def order(self, deg, n):
        orig = torch.empty(max(n, 1), dtype=torch.int32, device=self.dev)
        rel = torch.empty(max(n, 1), dtype=torch.int32, device=self.dev)
        self.L.call("tc_shard_order", self.L.ptr(deg), int(n), self.L.ptr(orig), self.L.ptr(rel), self.L.stream())
        return orig[:n], rel[:n]

    def orient(self, ukeys, relabel, n):
        k = int(ukeys.numel())
        lohi = torch.empty((max(k, 1), 2), dtype=torch.int32, device=self.dev)
        eff = torch.zeros(max(n, 1), dtype=torch.int32, device=self.dev)
        self.L.call("tc_shard_orient", self.L.ptr(ukeys), k, self.L.ptr(relabel), self.L.ptr(lohi), self.L.ptr(eff),
                    self.L.stream())
        return lohi[:k], eff[:n]

    def predsum(self, lohi, effdeg, n):
        c = torch.zeros(max(n, 1), dtype=torch.int64, device=self.dev)
        self.L.call("tc_shard_predsum", self.L.ptr(lohi), int(lohi.shape[0]), self.L.ptr(effdeg), self.L.ptr(c),
                    self.L.stream())
        return c[:n]

    def balanced(self, costs, n, P):
        b = torch.empty(P + 1, dtype=torch.int64, device=self.dev)
        self.L.call("tc_balanced_bounds", self.L.ptr(costs), 0, int(n), int(P), self.L.ptr(b), self.L.stream())
        return b.cpu().numpy()

    def route(self, lohi, bounds, P):
        k = int(lohi.shape[0])
        out = torch.empty((max(k, 1), 2), dtype=torch.int32, device=self.dev)
        counts = np.zeros(P, np.int64)
        b = torch.as_tensor(np.asarray(bounds, np.int64)).to(self.dev)
        self.L.call("tc_shard_route", self.L.ptr(lohi), k, self.L.ptr(b), int(P), self.L.ptr(out),
                    counts.ctypes.data_as(ctypes.c_void_p), self.L.stream())
        return out[:k], counts

    def csr(self, lohi, lo, nrow):
        k = int(lohi.shape[0])
        indptr = torch.empty(nrow + 1, dtype=torch.int64, device=self.dev)
        indices = torch.empty(k + 4, dtype=torch.int32, device=self.dev)  # +4: 16-byte chunk reads
        self.L.call("tc_shard_csr", self.L.ptr(lohi), k, int(lo), int(nrow), self.L.ptr(indptr), self.L.ptr(indices),
                    self.L.stream())
        return indptr, indices[:k]

    def pool(self, indptr, indices):
        nrow = int(indptr.numel()) - 1
        pip = torch.empty(nrow + 1, dtype=torch.int64, device=self.dev)
        buf = torch.empty(POOL_HEAD + int(indices.numel()) + 3 * nrow + 4, dtype=torch.int32, device=self.dev)
        pool = buf[POOL_HEAD:]
        self.L.call("tc_shard_pool", self.L.ptr(indptr), self.L.ptr(indices), nrow, self.L.ptr(pip),
                    self.L.ptr(pool), self.L.stream())
        return pip, pool

    def engine_cost_acc(self, indptr, indices, n):
        acc = torch.zeros(max(n, 1), dtype=torch.int64, device=self.dev)
        self.L.call("tc_shard_engine_cost", self.L.ptr(indptr), self.L.ptr(indices), int(indptr.numel()) - 1,
                    int(SEG_WEIGHT), self.L.ptr(acc), self.L.stream())
        return acc[:n]

    def engine_cost(self, acc, effdeg, n, tab_weight=1, send_weight=0):
        c = torch.empty(max(n, 1), dtype=torch.int64, device=self.dev)
        self.L.call("tc_shard_engine_cost_fin", self.L.ptr(acc), self.L.ptr(effdeg), int(n), int(tab_weight),
                    int(send_weight), self.L.ptr(c), self.L.stream())
        return c[:n]

    # -- count --
    def send_sizes(self, sh, P, rank):
        # a property of the partitioned graph (like the engine plan): computed
        # at the first count of a shard
        hit = sh.cache.get(("send_sizes", P, rank))
        if hit is not None:
            return hit
        plen = ctypes.c_int64()
        self.L.call("tc_shard_send_plan_len", sh.hi - sh.lo, int(P), ctypes.byref(plen))
        sizes = torch.empty(plen.value, dtype=torch.int64, device=self.dev)  # sizes + the pack's block plan
        host = np.zeros(3 * P, np.int64)
        b = sh.cache.get("bounds_dev")
        if b is None:
            b = sh.cache["bounds_dev"] = torch.as_tensor(np.asarray(sh.bounds, np.int64)).to(self.dev)
        self.L.call("tc_shard_send_sizes", self.L.ptr(sh.indptr), self.L.ptr(sh.indices), sh.hi - sh.lo,
                    self.L.ptr(sh.pool_indptr), self.L.ptr(b), int(P), int(rank), self.L.ptr(sizes),
                    host.ctypes.data_as(ctypes.c_void_p), self.L.stream())
        sh.cache[("send_sizes", P, rank)] = (sizes, host.reshape(3, P))
        return sizes, host.reshape(3, P)

    def send_pack(self, sh, P, rank, sizes_dev, nl, nw):
        lens = torch.empty(max(nl, 1), dtype=torch.int32, device=self.dev)
        ids = torch.empty(max(nw, 4), dtype=torch.int32, device=self.dev)
        t0 = self._tic()
        self.L.call("tc_shard_send_pack", self.L.ptr(sh.indptr), self.L.ptr(sh.indices), sh.hi - sh.lo,
                    self.L.ptr(sh.pool_indptr), self.L.ptr(sh.pool), self.L.ptr(sh.cache["bounds_dev"]), int(P),
                    int(rank), self.L.ptr(sizes_dev), self.L.ptr(lens), self.L.ptr(ids), self.L.stream())
        self._toc(t0, label="pack")
        return lens[:nl], ids[:nw]

    def recv_pool(self, nw):
        buf = torch.empty(POOL_HEAD + nw + 4, dtype=torch.int32, device=self.dev)
        buf[:POOL_HEAD].fill_(INT32_MAX)
        return buf, buf[POOL_HEAD: POOL_HEAD + nw]

    def _streams(self):
        st = getattr(self, "_st", None)
        if st is None:
            # planning (index + tier lists; it synchronises its own stream) and
            # engine runs go to side streams, so neither holds back the
            # collectives issued on the current stream
            st = self._st = (torch.cuda.Stream(device=self.dev), torch.cuda.Stream(device=self.dev),
                             torch.cuda.Stream(device=self.dev))
            self._turn = 0
        if self.timing:
            # measurement mode: everything on the current stream, so the event
            # brackets do not overlap and their sum is the rank's device work
            cur = torch.cuda.current_stream(self.dev)
            return (cur, cur, cur)
        return st

    def _plan(self, sh, row_len, pool):
        """tc_shard_index + tc_plan_middle over padded rows (row_len, pool):
        owners = the shard's range, tables = the shard's lists."""
        L = self.L
        nx = sh.hi - sh.lo
        nrow = int(row_len.numel())
        pip = torch.empty(nrow + 1, dtype=torch.int64, device=self.dev)
        rip = torch.empty(nx + 1, dtype=torch.int64, device=self.dev)
        cap = max(int(pool.numel()), 1)
        rseg = torch.empty(2 * cap, dtype=torch.int32, device=self.dev)
        rcost = torch.empty(nx + 1, dtype=torch.int64, device=self.dev)
        L.call("tc_shard_index", L.ptr(row_len), nrow, L.ptr(pool), int(pool.numel()), sh.lo, sh.hi, L.ptr(sh.indptr),
               L.ptr(pip),
               L.ptr(rip), L.ptr(rseg), L.ptr(rcost), None, L.stream())
        h = ctypes.c_void_p()
        L.call("tc_plan_middle", L.ptr(sh.indptr), L.ptr(sh.indices), L.ptr(rip), L.ptr(rseg), L.ptr(rcost),
               L.ptr(pool), 1, nx, 0, nx, None, 1, ctypes.byref(h), L.stream())
        from .distributed import _PlanHandle
        return _PlanHandle(h, (pip, rip, rseg, rcost, pool, row_len))

    def _launch(self, plan):
        """One engine run of a plan on a run stream; returns its output.
        Consecutive runs alternate between two streams, so a run's tail (the
        last chunks of its hubs) overlaps the start of the next one."""
        st = self._streams()
        self._turn ^= 1
        run_s = st[1 + self._turn]
        run_s.wait_stream(st[0])  # the plan was built on the plan stream
        with torch.cuda.stream(run_s):
            o = torch.empty(1, dtype=torch.int64, device=self.dev)
            t0 = self._tic(run_s)
            self.L.call("tc_plan_run", plan.handle, self.L.ptr(o), self.L.stream())
            self._toc(t0, run_s)
        return o

    def start_local(self, sh):
        """Engine run over the shard's own lists (plan cached on the shard)."""
        plan = sh.cache.get("local_plan")
        if plan is None:
            plan_s = self._streams()[0]
            plan_s.wait_stream(torch.cuda.current_stream(self.dev))
            with torch.cuda.stream(plan_s):
                row_len = (sh.indptr[1:] - sh.indptr[:-1]).to(torch.int32).contiguous()
                plan = sh.cache["local_plan"] = self._plan(sh, row_len, sh.pool)
        return self._launch(plan), plan

    def count_received(self, sh, row_len, pool, key=None):
        """Index + plan the received padded lists on the plan stream (after
        the current stream, which their transfer completed on), run them on
        a run stream.  Returns (out, plan): keep the plan until finish.

        key names the exchange round: a round delivers lists of the same
        structure at every count of a partitioned graph (the pack is
        deterministic), so the per-owner offsets, the cost prefix and the
        engine plan (all O(owned nodes)) are kept on the shard after the
        first count; later counts only scatter the segments of the fresh
        lists (tc_shard_index_emit) and point the plan at them."""
        L = self.L
        plan_s = self._streams()[0]
        plan_s.wait_stream(torch.cuda.current_stream(self.dev))
        hit = sh.cache.get(("recv_plan", key)) if key is not None else None
        with torch.cuda.stream(plan_s):
            t0 = self._tic(plan_s)
            if hit is None or hit[1] != (int(row_len.numel()), int(pool.numel())):
                plan = self._plan(sh, row_len, pool)
                if key is not None:
                    sh.cache[("recv_plan", key)] = (plan, (int(row_len.numel()), int(pool.numel())))
            else:
                plan = hit[0]
                nrow = int(row_len.numel())
                pip = torch.empty(nrow + 1, dtype=torch.int64, device=self.dev)
                rseg = torch.empty(2 * max(int(pool.numel()), 1), dtype=torch.int32, device=self.dev)
                rip = plan.keep[1]
                L.call("tc_shard_index_emit", L.ptr(row_len), nrow, L.ptr(pool), int(pool.numel()), sh.lo, sh.hi, L.ptr(rip),
                       L.ptr(pip),
                       L.ptr(rseg), L.stream())
                L.call("tc_plan_rebind", plan.handle, L.ptr(rseg), L.ptr(pool))
                # the plan's handle keeps the offsets and costs; this count's arrays live until finish
                plan.keep = (pip, rip, rseg, plan.keep[3], pool, row_len)
            self._toc(t0, plan_s, "index")
        return self._launch(plan), plan

    def release_received(self, plan):
        """Drops a received round's arrays from its (kept) plan once the
        count has finished: between counts a rank holds only its shard and
        the O(owned nodes) offsets, costs and plan of each round."""
        k = plan.keep
        plan.keep = (None, k[1], None, k[3], None, None)

    def finish(self, outs):
        """Sum of the run outputs, read after the run stream's work."""
        for st in self._streams()[1:]:
            torch.cuda.current_stream(self.dev).wait_stream(st)
        return int(sum(int(o.item()) for o in outs))

# ------------------------------------------------------------------ collectives

# Requests a rank generator yields:
#   ("allreduce", tensor, "sum" | "max" | "min")          -> reduced tensor
#   ("a2a", send, counts)  (send grouped by peer along dim 0, counts[P] rows)
#                                                        -> (recv, recv_counts)
#   ("a2a_start", send, counts, recv_counts)               -> handle
#   ("wait", handle)                                       -> recv


def run_dist(gen, group=None):
    """Drives one rank's generator over torch.distributed."""
    import torch.distributed as dist

    ops = {"sum": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN}
    P = dist.get_world_size(group)
    res = None
    while True:
        try:
            req = gen.send(res)
        except StopIteration as stop:
            return stop.value
        kind = req[0]
        if kind == "allreduce":
            t = req[1]
            dist.all_reduce(t, op=ops[req[2]], group=group)
            res = t
        elif kind == "a2a":
            send, counts = req[1], np.asarray(req[2], np.int64)
            ct = torch.as_tensor(counts).to(send.device)
            rc = torch.empty(P, dtype=torch.int64, device=send.device)
            dist.all_to_all_single(rc, ct, group=group)
            rcounts = rc.cpu().numpy()
            recv = torch.empty((int(rcounts.sum()),) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
            dist.all_to_all_single(recv, send.contiguous(), output_split_sizes=rcounts.tolist(),
                                   input_split_sizes=counts.tolist(), group=group)
            res = (recv, rcounts)
        elif kind == "a2a_start":
            send, counts, rcounts = req[1], np.asarray(req[2], np.int64), np.asarray(req[3], np.int64)
            recv = req[4] if len(req) > 4 and req[4] is not None else torch.empty(
                (int(rcounts.sum()),) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
            work = dist.all_to_all_single(recv, send.contiguous(), output_split_sizes=rcounts.tolist(),
                                          input_split_sizes=counts.tolist(), group=group, async_op=True)
            res = (work, recv)
        elif kind == "wait":
            work, recv = req[1]
            work.wait()
            res = recv
        else:
            raise ValueError(f"unknown collective {kind}")


def ops_of(gen):
    """The ops object a rank generator was started with (emulation timing)."""
    try:
        return gen.gi_frame.f_locals.get("ops")
    except AttributeError:
        return None


class CComm:
    """A communicator of the C ABI's NCCL layer (tc_nccl_*, tc_allreduce,
    tc_exchange): the path a reference-side binding drives without
    torch.distributed."""

    DT = {torch.uint8: 0, torch.int32: 1, torch.int64: 2}
    OP = {"sum": 0, "max": 1, "min": 2}

    def __init__(self, uid: bytes, nranks: int, rank: int):
        from . import _lib

        self.L, self.P, self.rank = _lib, nranks, rank
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(uid, 128)
        _lib.call("tc_nccl_init_rank", buf, int(nranks), int(rank), ctypes.byref(h))
        self.h = h

    @staticmethod
    def unique_id() -> bytes:
        from . import _lib

        buf = ctypes.create_string_buffer(128)
        _lib.call("tc_nccl_unique_id", buf)
        return buf.raw

    def close(self):
        if self.h:
            self.L.lib().tc_nccl_free(self.h)
            self.h = None

    def allreduce(self, t, op):
        self.L.call("tc_allreduce", self.L.ptr(t), int(t.numel()), self.DT[t.dtype], self.OP[op], self.h,
                    self.L.stream())
        return t

    def exchange(self, send, counts, rcounts, recv=None):
        """all-to-all-v along dim 0 (counts in rows)."""
        row = int(np.prod(send.shape[1:])) if send.dim() > 1 else 1
        if recv is None:
            recv = torch.empty((int(np.sum(rcounts)),) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
        sc = (np.asarray(counts, np.int64) * row).astype(np.int64)
        rc = (np.asarray(rcounts, np.int64) * row).astype(np.int64)
        self.L.call("tc_exchange", self.L.ptr(send.contiguous()), sc.ctypes.data_as(ctypes.c_void_p),
                    self.L.ptr(recv), rc.ctypes.data_as(ctypes.c_void_p), self.DT[send.dtype], self.P, self.h,
                    self.L.stream())
        return recv


def run_capi(gen, comm: CComm):
    """Drives one rank's generator over the C ABI's NCCL layer."""
    res = None
    while True:
        try:
            req = gen.send(res)
        except StopIteration as stop:
            return stop.value
        kind = req[0]
        if kind == "allreduce":
            res = comm.allreduce(req[1], req[2])
        elif kind == "a2a":
            send, counts = req[1], np.asarray(req[2], np.int64)
            ct = torch.as_tensor(counts).to(send.device)
            rc = comm.exchange(ct, np.ones(comm.P, np.int64), np.ones(comm.P, np.int64))
            rcounts = rc.cpu().numpy()
            res = (comm.exchange(send, counts, rcounts), rcounts)
        elif kind == "a2a_start":  # stream-ordered: the wait is a no-op for the host
            into = req[4] if len(req) > 4 else None
            res = comm.exchange(req[1], req[2], req[3], into)
        elif kind == "wait":
            res = req[1]
        else:
            raise ValueError(f"unknown collective {kind}")


def emulate(gens, timed=False, busy=None, labels=None):
    """Runs P rank generators in lockstep in this process (one device): every
    collective is performed once all ranks have reached it.  With timed=True
    each rank's device work between collectives is bracketed by CUDA events
    (host gaps between its kernels included); returns (results, per-rank
    device ms).  busy (a list of P zeros) collects, per rank, the event
    brackets of its own kernels (ShardOps.busy_ms: pack, receive index,
    engine runs) -- the measure bench.py's N-GPU run feeds to the
    refinement."""
    P = len(gens)
    res = [None] * P
    done = [False] * P
    out = [None] * P
    ms = [0.0] * P
    pending = {}
    ticket = 0
    while not all(done):
        reqs = [None] * P
        for r in range(P):
            if done[r]:
                continue
            if timed:
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
            o = ops_of(gens[r]) if busy is not None else None
            try:
                reqs[r] = gens[r].send(res[r])
            except StopIteration as stop:
                done[r] = True
                out[r] = stop.value
            if o is not None and getattr(o, "timing", False):
                lab = {}
                busy[r] += o.busy_ms(lab)
                if labels is not None:
                    for k, v in lab.items():
                        labels[r][k] = labels[r].get(k, 0.0) + v
            if timed:
                # the segment's side-stream work (engine runs, planning) is
                # counted with it: per-rank time is serialised (no overlap
                # between the exchange and the local engine)
                for st in getattr(ops_of(gens[r]), "_st", None) or ():
                    torch.cuda.current_stream().wait_stream(st)
                e.record()
                torch.cuda.synchronize()
                ms[r] += s.elapsed_time(e)
        live = [r for r in range(P) if not done[r]]
        if not live:
            break
        kinds = {reqs[r][0] for r in live}
        if len(kinds) != 1 or len(live) != P:
            raise RuntimeError(f"ranks diverged at a collective: {kinds}, live {live}")
        kind = kinds.pop()
        if kind == "allreduce":
            ts = [reqs[r][1] for r in range(P)]
            op = reqs[0][2]
            acc = ts[0].clone()
            for t in ts[1:]:
                acc = acc + t if op == "sum" else (torch.maximum(acc, t) if op == "max" else torch.minimum(acc, t))
            for r in range(P):
                ts[r].copy_(acc)
                res[r] = ts[r]
        elif kind in ("a2a", "a2a_start"):
            sends = [reqs[r][1] for r in range(P)]
            counts = [np.asarray(reqs[r][2], np.int64) for r in range(P)]
            offs = [np.concatenate([[0], np.cumsum(c)]) for c in counts]
            for r in range(P):
                parts = [sends[s][int(offs[s][r]): int(offs[s][r + 1])] for s in range(P)]
                rc = np.array([int(counts[s][r]) for s in range(P)], np.int64)
                recv = torch.cat(parts) if parts else sends[r][:0]
                if kind == "a2a":
                    res[r] = (recv, rc)
                else:
                    into = reqs[r][4] if len(reqs[r]) > 4 else None
                    if into is not None and recv.numel():
                        into.copy_(recv)
                        recv = into
                    ticket += 1
                    pending[ticket] = recv
                    res[r] = ("emu", ticket)
        elif kind == "wait":
            for r in range(P):
                res[r] = pending.pop(reqs[r][1][1])
        else:
            raise ValueError(f"unknown collective {kind}")
    return out, ms


# ------------------------------------------------------------------ the rank steps

def build_gen(pairs, pos_base, P, rank, cost="predsum", ops=None, keep_maps=False):
    """One rank of the sharded build (steps 1-5).  pairs: this rank's raw
    slice, int32 (k, 2) on the rank's device; pos_base: index of its first
    pair in the whole raw list.  Returns a ShardGraph."""
    ops = ops or ShardOps()
    dev = pairs.device if isinstance(pairs, torch.Tensor) else None
    # 1. labels
    mn, mx = ops.minmax(pairs) if pairs.shape[0] else (2**31 - 1, -1)
    t = torch.tensor([mx, -mn], dtype=torch.int64, device=dev)
    t = yield ("allreduce", t, "max")
    gmax, gmin = int(t[0]), -int(t[1])
    if gmax >= 0 and gmin < 0:  # graph.py:87-88
        raise ValueError("negative node id in edge list")
    K = gmax + 1 if gmax >= 0 else 0
    present, first = ops.label_scan(pairs, pos_base, K)
    present = yield ("allreduce", present, "max")
    first = yield ("allreduce", first, "min")
    mp, n, dense = ops.relabel_map(present, first, K)
    del present, first
    # 2. dedup by hash of the canonical key
    keys, counts = ops.keys(pairs, None if dense else mp, P)
    del mp
    recv, _ = yield ("a2a", keys, counts)
    del keys
    ukeys = ops.dedup(recv, n)
    del recv
    # 3. degrees and the canonical order
    deg = ops.degrees(ukeys, n)
    deg = yield ("allreduce", deg, "sum")
    orig_ids, relabel = ops.order(deg, n)
    del deg
    # 4. orientation, out-degrees, the partition
    lohi, effdeg = ops.orient(ukeys, relabel, n)
    del ukeys
    effdeg = yield ("allreduce", effdeg, "sum")
    mt = torch.tensor([int(lohi.shape[0])], dtype=torch.int64, device=dev)
    mt = yield ("allreduce", mt, "sum")
    m = int(mt[0])
    c = ops.predsum(lohi, effdeg, n)
    c = yield ("allreduce", c, "sum")
    bounds = ops.balanced(c, n, P)
    weights = c
    # 5. the shard: pairs to the owner of lo
    routed, counts = ops.route(lohi, bounds, P)
    del lohi
    mine, _ = yield ("a2a", routed, counts)
    del routed
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    indptr, indices = ops.csr(mine, lo, hi - lo)
    del mine
    if cost == "engine":
        # re-balance by the middle-vertex engine's own per-owner cost and move
        # the rows whose owner changed (contiguous ranges: concatenating the
        # pieces in source-rank order keeps rows ascending)
        acc = ops.engine_cost_acc(indptr, indices, n)
        acc = yield ("allreduce", acc, "sum")
        ec = ops.engine_cost(acc, effdeg, n, TAB_WEIGHT, SEND_WEIGHT)
        del acc
        nb = ops.balanced(ec, n, P)
        weights = ec
        indptr, indices = yield from _repartition(indptr, indices, lo, hi, nb, P, dev)
        bounds = nb
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    elif cost != "predsum":
        raise ValueError(f"unknown partition cost {cost!r} (predsum or engine)")
    del effdeg
    pip, pool = ops.pool(indptr, indices)
    sh = ShardGraph(lo, hi, n, m, np.asarray(bounds, np.int64), indptr, indices, pip, pool)
    # the per-node weights the partition was cut by (replicated, O(n)): the
    # measured refinement (rebalance_gen) rescales them
    sh.cache["weights"] = weights
    if keep_maps:
        sh.relabel, sh.orig_ids = relabel, orig_ids
    return sh


def _repartition(indptr, indices, lo, hi, nb, P, dev):
    """Rows [lo, hi) redistributed to the ranges of bounds nb."""
    lens = (indptr[1:] - indptr[:-1]).to(torch.int32)
    rc = np.zeros(P, np.int64)
    ic = np.zeros(P, np.int64)
    # row offsets at the new bounds only (2 P entries, not the whole offsets array)
    cuts = np.array([[min(max(int(nb[j]), lo), hi) - lo, min(max(int(nb[j + 1]), lo), hi) - lo] for j in range(P)],
                    np.int64)
    at = indptr[torch.as_tensor(cuts.reshape(-1)).to(indptr.device)].cpu().numpy().reshape(P, 2)
    for j in range(P):
        if cuts[j, 0] < cuts[j, 1]:
            rc[j] = cuts[j, 1] - cuts[j, 0]
            ic[j] = int(at[j, 1] - at[j, 0])
    rl, _ = yield ("a2a", lens.contiguous(), rc)
    ri, _ = yield ("a2a", indices.contiguous(), ic)
    nip = torch.zeros(int(rl.numel()) + 1, dtype=torch.int64, device=dev)
    if rl.numel():
        nip[1:] = torch.cumsum(rl.to(torch.int64), 0)
    return nip, ri


def rebalance_gen(sh: ShardGraph, P, rank, busy_ms, ops=None):
    """Measured refinement of the partition (the cost-function partition of
    partitioning.py:79-141 with the cost taken from a run instead of a
    model): every rank reports the device time of its last count, the node
    weights of rank r's range are scaled by time_r / weight_r (so the weight
    of a range is the time it took), the bounds are re-balanced on the scaled
    weights and the rows whose owner changed move (one all_to_all of row
    lengths and one of ids).  Returns the new ShardGraph; the old one is
    consumed."""
    ops = ops or ShardOps()
    dev = sh.indptr.device
    w = sh.cache.get("weights")
    if w is None:
        raise ValueError("the shard carries no partition weights")
    t = torch.zeros(P, dtype=torch.int64, device=dev)
    t[rank] = max(1, int(round(1e3 * float(busy_ms))))  # microseconds
    t = yield ("allreduce", t, "sum")
    b = torch.as_tensor(np.asarray(sh.bounds, np.int64)).to(dev)
    wf = w.to(torch.float64)
    pre = torch.cat([torch.zeros(1, dtype=torch.float64, device=dev), torch.cumsum(wf, 0)])
    tot = pre[b[1:]] - pre[b[:-1]]
    scale = t.to(torch.float64) / torch.clamp(tot, min=1.0)
    owner = torch.bucketize(torch.arange(sh.n, device=dev), b[1:-1].contiguous(), right=True)
    wf = wf * scale[owner]
    # integer weights again (tc_balanced_bounds), ~2^44 in total
    wn = torch.clamp((wf * (float(1 << 44) / max(float(wf.sum()), 1.0))).round(), min=0).to(torch.int64)
    del wf, pre, owner
    nb = ops.balanced(wn, sh.n, P)
    indptr, indices = yield from _repartition(sh.indptr, sh.indices, sh.lo, sh.hi, nb, P, dev)
    lo, hi = int(nb[rank]), int(nb[rank + 1])
    pip, pool = ops.pool(indptr, indices)
    out = ShardGraph(lo, hi, sh.n, sh.m, np.asarray(nb, np.int64), indptr, indices, pip, pool, sh.relabel, sh.orig_ids)
    out.cache["weights"] = wn
    sh.cache.clear()
    return out


def _phase(prof, name, t0):
    """Profiling hook (prof dict given): device-synchronised phase times."""
    if prof is None:
        return t0
    torch.cuda.synchronize()
    t = time.perf_counter()
    prof[name] = prof.get(name, 0.0) + 1e3 * (t - t0)
    return t


def count_gen(sh: ShardGraph, P, rank, ops=None, round_words=1 << 28, met=None, prof=None):
    """One rank of the count (steps 6-8); returns (total, RankMetrics).
    round_words bounds the padded ids a rank receives per exchange round.
    prof (a dict, profiling only) collects synchronised per-phase times."""
    ops = ops or ShardOps()
    dev = sh.indptr.device
    tp = _phase(prof, "start", time.perf_counter()) if prof is not None else None
    met = met or RankMetrics(rank=rank, nranks=P)
    met.partition_bytes = WORD_BYTES * ((sh.hi - sh.lo) + 1 + sh.m_local)
    outs, keep = [], []
    # 6. local lists first: the engine runs (side stream) while the exchange
    # is in flight
    if sh.hi > sh.lo and sh.m_local:
        o, plan = ops.start_local(sh)
        outs.append(o)
    tp = _phase(prof, "local", tp)
    # 7. the exchange: sizes, packed messages, bounded rounds
    sizes_dev, sizes = ops.send_sizes(sh, P, rank)
    lists, words, full = sizes[0], sizes[1], sizes[2]
    met.data_msgs_to = lists.astype(np.int64).copy()
    met.data_msgs_sent = int(lists.sum())
    met.completion_msgs_sent = P - 1
    met.bytes_sent = WORD_BYTES * (2 * int(lists.sum()) + int(full.sum()) + (P - 1))
    xkey = ("xplan", P, rank, round_words)
    xplan = sh.cache.get(xkey) if hasattr(sh, "cache") else None
    if xplan is None:
        # what every peer sends here, and the round structure: static for a
        # partitioned graph, exchanged at its first count
        st = torch.as_tensor(np.stack([lists, words], 1).astype(np.int64)).to(dev)
        rsz, _ = yield ("a2a", st, np.ones(P, np.int64))
        rsz = rsz.cpu().numpy() if isinstance(rsz, torch.Tensor) else np.asarray(rsz)
        rlists, rwords = rsz[:, 0], rsz[:, 1]
        # rounds over sender ranks: in a round the ranks of a consecutive
        # group send all their messages and every rank above them receives;
        # a group closes once the largest volume a rank would receive in it
        # would pass round_words -- the same grouping on every rank (from the
        # replicated P x P volume matrix)
        hv = np.zeros((P, P), np.int64)
        hv[rank, :rank] = np.asarray(rwords, np.int64)[:rank]
        vol = torch.as_tensor(hv.reshape(-1)).to(dev)
        vol = yield ("allreduce", vol, "sum")
        vol = (vol.cpu().numpy() if isinstance(vol, torch.Tensor) else np.asarray(vol)).reshape(P, P)
        rounds, cur, acc = [], [], np.zeros(P, np.int64)
        for s_ in range(P - 1):
            if cur and int((acc + vol[:, s_]).max()) > round_words:
                rounds.append(cur)
                cur, acc = [], np.zeros(P, np.int64)
            cur.append(s_)
            acc = acc + vol[:, s_]
        if cur:
            rounds.append(cur)
        xplan = (rlists, rwords, rounds)
        if hasattr(sh, "cache"):
            sh.cache[xkey] = xplan
    rlists, rwords, rounds = xplan
    lens, ids = ops.send_pack(sh, P, rank, sizes_dev, int(lists.sum()), int(words.sum()))
    tp = _phase(prof, "pack", tp)
    met.wire_bytes = int(4 * (lists.sum() + words.sum()) + 16 * P)
    pending = None
    for ri, rd in enumerate(rounds):
        sl, sw = np.zeros(P, np.int64), np.zeros(P, np.int64)
        rl, rw = np.zeros(P, np.int64), np.zeros(P, np.int64)
        if rank in rd:  # this rank's turn: all its messages, grouped by destination
            sl[rank + 1:], sw[rank + 1:] = lists[rank + 1:], words[rank + 1:]
            send_l, send_w = lens, ids
        else:
            send_l, send_w = lens[:0], ids[:0]
        for s_ in rd:
            if s_ < rank:
                rl[s_], rw[s_] = rlists[s_], rwords[s_]
        buf, rpool = ops.recv_pool(int(rw.sum()))
        h_l = yield ("a2a_start", send_l, sl, rl, None)
        h_w = yield ("a2a_start", send_w, sw, rw, rpool)
        tp = _phase(prof, "round_setup", tp)
        if pending is not None:  # count the previous round while this one is in flight
            o, plan = ops.count_received(sh, pending[0], pending[1], key=(xkey, pending[3]))
            outs.append(o)
            keep.append((plan, pending))
            tp = _phase(prof, "received", tp)
        r_len = yield ("wait", h_l)
        r_ids = yield ("wait", h_w)
        if r_ids.numel() and r_ids.data_ptr() != rpool.data_ptr():
            rpool.copy_(r_ids)
        pending = (r_len.to(torch.int32).contiguous(), rpool, buf, ri) if int(rl.sum()) else None
    tp = _phase(prof, "round_setup", tp)
    if pending is not None:
        o, plan = ops.count_received(sh, pending[0], pending[1], key=(xkey, pending[3]))
        outs.append(o)
        keep.append((plan, pending))
        tp = _phase(prof, "received", tp)
    part = ops.finish(outs)
    rel = getattr(ops, "release_received", None)
    if rel is not None:
        for plan, _ in keep:
            rel(plan)
    del keep
    met.triangles = part
    tot = torch.tensor([part], dtype=torch.int64, device=dev)
    tot = yield ("allreduce", tot, "sum")  # 8.
    return int(tot[0]), met


_MET_FIELDS = ("triangles", "data_msgs_sent", "bytes_sent", "requests_sent", "completion_msgs_sent",
               "tasks_executed", "partition_bytes", "wire_bytes")


def gather_metrics_gen(met: RankMetrics, P, rank, dev=None, busy_ms=0.0):
    """Every rank's RankMetrics on every rank (the per-rank rows of the
    reference's run CSV, metrics.py:49-116, from a real N-rank run): one
    all-reduce of an int64 matrix in which rank r fills row r (counters,
    busy time in microseconds, data_msgs_to)."""
    k = len(_MET_FIELDS) + 1
    row = np.zeros((P, k + P), np.int64)
    row[rank, : k - 1] = [int(getattr(met, f)) for f in _MET_FIELDS]
    row[rank, k - 1] = int(round(1e3 * float(busy_ms)))
    row[rank, k:] = np.asarray(met.data_msgs_to, np.int64)
    t = torch.as_tensor(row.reshape(-1))
    t = t.to(dev) if dev is not None else t
    t = yield ("allreduce", t, "sum")
    a = (t.cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)).reshape(P, k + P)
    out = []
    for r in range(P):
        m = RankMetrics(rank=r, nranks=P)
        for i, f in enumerate(_MET_FIELDS):
            setattr(m, f, int(a[r, i]))
        m.busy_time = a[r, k - 1] / 1e6  # seconds
        m.data_msgs_to = a[r, k:].copy()
        out.append(m)
    return out


def run_record(total, mets, wall_s, graph="", seed=0, cost="predsum", suite="count"):
    """The reference's RunRecord (metrics.py:49-83) of one sharded count:
    algo "surrogate", backend "b200" (time cells are device seconds)."""
    from .metrics import RunRecord

    return RunRecord(algo="surrogate", ranks=len(mets), cost=cost, graph=graph, seed=seed, backend="b200",
                     wall_time=wall_s, total=total, rows=list(mets), suite=suite)


def shard_from_graph(g, bounds, rank, ops=None) -> ShardGraph:
    """Rank `rank`'s ShardGraph cut out of a whole (replicated) Graph: its
    forward lists and the engine's padded copy of them.  For callers of the
    reference-style API that already hold the graph on every rank
    (distributed.count_space_surrogate_dist)."""
    ops = ops or ShardOps()
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    e0, e1 = int(g.eff_indptr[lo]), int(g.eff_indptr[hi])
    indptr = (g.eff_indptr[lo: hi + 1] - e0).contiguous()
    buf = torch.zeros(e1 - e0 + 4, dtype=torch.int32, device=indptr.device)  # +4: 16-byte chunk reads
    buf[: e1 - e0] = g.eff_indices[e0:e1]
    indices = buf[: e1 - e0]
    pip, pool = ops.pool(indptr, indices)
    return ShardGraph(lo, hi, int(g.n), int(g.m), np.asarray(bounds, np.int64), indptr, indices, pip, pool)


def slice_of(raw, P, rank):
    """Rank r's slice of a raw pair list and its first pair's index."""
    m = int(raw.shape[0])
    a, b = m * rank // P, m * (rank + 1) // P
    return raw[a:b], a


# ------------------------------------------------------------------ entry points

def build_sharded(pairs, pos_base, group=None, cost="predsum", ops=None, keep_maps=False):
    """The sharded build on this rank (torch.distributed initialised)."""
    import torch.distributed as dist

    P, rank = dist.get_world_size(group), dist.get_rank(group)
    return run_dist(build_gen(pairs, pos_base, P, rank, cost, ops, keep_maps), group)


def count_sharded(sh: ShardGraph, group=None, ops=None, round_words=1 << 28):
    """The sharded surrogate count on this rank; returns (total, RankMetrics)."""
    import torch.distributed as dist

    P, rank = dist.get_world_size(group), dist.get_rank(group)
    return run_dist(count_gen(sh, P, rank, ops, round_words), group)


def gather_metrics(met: RankMetrics, group=None, busy_ms=0.0, device=None):
    """All ranks' RankMetrics on this rank (torch.distributed initialised)."""
    import torch.distributed as dist

    P, rank = dist.get_world_size(group), dist.get_rank(group)
    return run_dist(gather_metrics_gen(met, P, rank, device, busy_ms), group)


def rebalance_sharded(sh: ShardGraph, busy_ms, group=None, ops=None):
    """Measured refinement of the partition on this rank (see rebalance_gen)."""
    import torch.distributed as dist

    P, rank = dist.get_world_size(group), dist.get_rank(group)
    return run_dist(rebalance_gen(sh, P, rank, busy_ms, ops), group)


def emulate_rebalance(shards, busy_ms, ops=None):
    """All P ranks of the measured refinement in this process."""
    P = len(shards)
    res, _ = emulate([rebalance_gen(sh, P, r, busy_ms[r], ops) for r, sh in enumerate(shards)])
    return res


def emulate_build(raw, P, cost="predsum", ops=None, keep_maps=False, timed=False):
    """All P ranks of the sharded build in this process; returns
    ([ShardGraph], per-rank device ms)."""
    gens = []
    for r in range(P):
        sl, base = slice_of(raw, P, r)
        gens.append(build_gen(sl.contiguous(), base, P, r, cost, ops, keep_maps))
    return emulate(gens, timed)


def emulate_count(shards, ops=None, round_words=1 << 28, timed=False, profs=None, busy=None, labels=None):
    """All P ranks of the sharded count in this process; returns
    (total, [RankMetrics], per-rank device ms)."""
    P = len(shards)
    rops = list(ops) if isinstance(ops, (list, tuple)) else [ops] * P  # one ops object per rank, or a shared one
    if busy is not None and ops is None:  # one timed ops object per rank
        rops = [ShardOps() for _ in range(P)]
    if busy is not None:
        for o in rops:
            if hasattr(o, "busy_ms"):
                o.timing = True
    res, ms = emulate([count_gen(sh, P, r, rops[r], round_words, prof=None if profs is None else profs[r])
                       for r, sh in enumerate(shards)], timed, busy, labels)
    return res[0][0], [x[1] for x in res], ms
