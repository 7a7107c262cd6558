"""Test-side helpers for the multi-rank path: a numpy implementation of the
per-rank primitives (restating scan_for_surrogate / surrogate_count_list,
_kernels.py:70-126) to drive distributed.surrogate_rank on CPU with gloo."""

import numpy as np
import torch


class NumpyOps:
    def records(self, shard, bounds, P, rank):
        ip = shard.indptr.numpy()
        ix = shard.indices.numpy()
        b = np.asarray(bounds, np.int64)
        recs = []
        for v in range(shard.lo, shard.hi):
            lst = ix[ip[v - shard.lo]: ip[v - shard.lo + 1]]
            owners = np.searchsorted(b, lst, side="right") - 1
            last = -1
            for j in owners.tolist():
                if j != rank and j != last:
                    recs.append((j, v))
                    last = j
        recs.sort(key=lambda t: t[0])  # stable: v ascending within dest
        counts = np.zeros(P, np.int64)
        for j, _ in recs:
            counts[j] += 1
        return torch.tensor([v for _, v in recs], dtype=torch.int32), counts

    def pack(self, shard, rec_v):
        ip = shard.indptr.numpy()
        ix = shard.indices.numpy()
        lens, ids = [], []
        for v in rec_v.tolist():
            lst = ix[ip[v - shard.lo]: ip[v - shard.lo + 1]]
            lens.append(len(lst))
            ids.extend(lst.tolist())
        return torch.tensor(lens, dtype=torch.int64), torch.tensor(ids, dtype=torch.int32)

    def count(self, shard, recv_len, recv_ids):
        ip = shard.indptr.numpy()
        ix = shard.indices.numpy()
        lo, hi = shard.lo, shard.hi

        def lst(u):
            return set(ix[ip[u - lo]: ip[u - lo + 1]].tolist())

        total = 0
        for v in range(lo, hi):  # local pairs (scan_for_surrogate)
            lv = lst(v)
            for u in lv:
                if lo <= u < hi:
                    total += len(lv & lst(u))
        off = 0
        ids = recv_ids.numpy()
        for ln in recv_len.tolist():  # received lists (surrogate_count_list)
            x = ids[off: off + ln]
            off += ln
            xs = set(x.tolist())
            for u in x.tolist():
                if lo <= u < hi:
                    total += len(xs & lst(u))
        return total


    # -- direct scheme (space_efficient.py:179-231) --
    def requests(self, shard, bounds, P, rank):
        ix = shard.indices.numpy()[: shard.m]
        rem = ix[ix >= shard.hi]
        ids, mult = np.unique(rem, return_counts=True)
        b = np.asarray(bounds, np.int64)
        owners = np.searchsorted(b, ids, side="right") - 1
        counts = np.bincount(owners, minlength=P).astype(np.int64)
        ref = np.bincount(owners, weights=mult, minlength=P).astype(np.int64)
        return (torch.as_tensor(ids.astype(np.int32)), torch.as_tensor(mult.astype(np.int64)), counts, ref)

    def count_direct(self, shard, req_ids, fetched_len, fetched_ids):
        ip = shard.indptr.numpy()
        ix = shard.indices.numpy()
        lo, hi = shard.lo, shard.hi
        lists = {}
        off = 0
        fids = fetched_ids.numpy()
        for u, ln in zip(req_ids.tolist(), fetched_len.tolist()):
            lists[u] = set(fids[off: off + ln].tolist())
            off += ln
        for v in range(lo, hi):
            lists[v] = set(ix[ip[v - lo]: ip[v - lo + 1]].tolist())
        total = 0
        for v in range(lo, hi):  # count_node_range(lo, hi), _kernels.py:40-52
            for u in lists[v]:
                total += len(lists[v] & lists[u])
        return total


def shard_from_arrays(eff_indptr, eff_indices, lo, hi):
    from paper_1406_5687_b200.distributed import Shard

    e0, e1 = int(eff_indptr[lo]), int(eff_indptr[hi])
    ip = torch.as_tensor(np.asarray(eff_indptr[lo: hi + 1], np.int64) - e0)
    ix = torch.as_tensor(np.asarray(eff_indices[e0:e1], np.int32))
    return Shard(lo, hi, ip, ix)
