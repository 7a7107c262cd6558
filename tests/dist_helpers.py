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


class NumpyShardOps:
    """numpy restatement of the sharded pipeline's per-rank device steps
    (paper_1406_5687_b200/sharded.py ShardOps, csrc/shard.cu), so the
    protocol -- collectives, rounds, bookkeeping -- runs on CPU with gloo."""

    HEAD = 512
    IMAX = 2**31 - 1

    @staticmethod
    def _np(t):
        return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)

    def minmax(self, pairs):
        p = self._np(pairs)
        return int(p.min()), int(p.max())

    def label_scan(self, pairs, base, K):
        p = self._np(pairs).astype(np.int64).reshape(-1, 2)
        present = np.zeros(K, np.uint8)
        first = np.full(K, 0x7F7F7F7F, np.int32)
        keep = p[:, 0] != p[:, 1]
        i = np.nonzero(keep)[0]
        a, b = p[keep, 0], p[keep, 1]
        present[a] = 1
        present[b] = 1
        np.minimum.at(first, a, (2 * (base + i)).astype(np.int32))
        np.minimum.at(first, b, (2 * (base + i) + 1).astype(np.int32))
        return torch.as_tensor(present), torch.as_tensor(first)

    def relabel_map(self, present, first, K):
        pr, fi = self._np(present), self._np(first)
        c = int(pr.sum())
        if c == K:
            return torch.arange(K, dtype=torch.int32), c, True
        key = np.where(pr > 0, fi.astype(np.int64), 2**32)
        order = np.argsort(key, kind="stable")[:c]
        mp = np.full(K, -1, np.int32)
        mp[order] = np.arange(c, dtype=np.int32)
        return torch.as_tensor(mp), c, False

    def keys(self, pairs, mp, P):
        p = self._np(pairs).astype(np.int64).reshape(-1, 2)
        p = p[p[:, 0] != p[:, 1]]
        if mp is not None:
            m = self._np(mp).astype(np.int64)
            p = m[p]
        k = (np.minimum(p[:, 0], p[:, 1]) << 32) | np.maximum(p[:, 0], p[:, 1])
        with np.errstate(over="ignore"):
            h = (k.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)) >> np.uint64(33)
        d = (h % np.uint64(P)).astype(np.int64)
        o = np.argsort(d, kind="stable")
        return torch.as_tensor(k[o]), np.bincount(d, minlength=P).astype(np.int64)

    def dedup(self, keys, n):
        return torch.as_tensor(np.unique(self._np(keys)))

    def degrees(self, ukeys, n):
        k = self._np(ukeys)
        return torch.as_tensor((np.bincount(k >> 32, minlength=n) + np.bincount(k & 0xFFFFFFFF, minlength=n))
                               .astype(np.int32))

    def order(self, deg, n):
        orig = np.argsort(self._np(deg), kind="stable").astype(np.int32)
        rel = np.empty(n, np.int32)
        rel[orig] = np.arange(n, dtype=np.int32)
        return torch.as_tensor(orig), torch.as_tensor(rel)

    def orient(self, ukeys, relabel, n):
        k = self._np(ukeys)
        r = self._np(relabel).astype(np.int64)
        a, b = r[k >> 32], r[k & 0xFFFFFFFF]
        lohi = np.stack([np.minimum(a, b), np.maximum(a, b)], 1).astype(np.int32)
        return torch.as_tensor(lohi), torch.as_tensor(np.bincount(lohi[:, 0], minlength=n).astype(np.int32))

    def predsum(self, lohi, effdeg, n):
        e = self._np(lohi).astype(np.int64)
        d = self._np(effdeg).astype(np.int64)
        c = np.zeros(n, np.int64)
        np.add.at(c, e[:, 1], d[e[:, 0]] + d[e[:, 1]])
        return torch.as_tensor(c)

    def balanced(self, costs, n, P):
        from oracle import oracle as O
        return np.asarray(O.balanced_bounds(self._np(costs).astype(np.int64), 0, n, P), np.int64)

    def route(self, lohi, bounds, P):
        e = self._np(lohi)
        d = np.searchsorted(np.asarray(bounds, np.int64), e[:, 0], side="right") - 1
        o = np.argsort(d, kind="stable")
        return torch.as_tensor(e[o]), np.bincount(d, minlength=P).astype(np.int64)

    def csr(self, lohi, lo, nrow):
        e = self._np(lohi).astype(np.int64)
        o = np.lexsort((e[:, 1], e[:, 0]))
        e = e[o]
        ip = np.zeros(nrow + 1, np.int64)
        ip[1:] = np.cumsum(np.bincount(e[:, 0] - lo, minlength=nrow))
        return torch.as_tensor(ip), torch.as_tensor(e[:, 1].astype(np.int32))

    def _padded(self, ip, ix):
        nrow = len(ip) - 1
        sz = (np.diff(ip) + 3) & ~3
        pip = np.zeros(nrow + 1, np.int64)
        pip[1:] = np.cumsum(sz)
        buf = np.full(self.HEAD + int(pip[-1]) + 4, self.IMAX, np.int32)
        for v in range(nrow):
            buf[self.HEAD + pip[v]: self.HEAD + pip[v] + ip[v + 1] - ip[v]] = ix[ip[v]: ip[v + 1]]
        return pip, buf

    def pool(self, indptr, indices):
        pip, buf = self._padded(self._np(indptr), self._np(indices))
        b = torch.as_tensor(buf)
        return torch.as_tensor(pip), b[self.HEAD:]

    def engine_cost_acc(self, indptr, indices, n):
        from paper_1406_5687_b200 import sharded as S
        ip, ix = self._np(indptr), self._np(indices).astype(np.int64)
        acc = np.zeros(n, np.int64)
        for v in range(len(ip) - 1):
            d = ip[v + 1] - ip[v]
            np.add.at(acc, ix[ip[v]: ip[v + 1]], d - np.arange(d) - 1 + S.SEG_WEIGHT)
        return torch.as_tensor(acc)

    def engine_cost(self, acc, effdeg, n, tab_weight=1, send_weight=0):
        a, d = self._np(acc), self._np(effdeg).astype(np.int64)
        return torch.as_tensor((np.where((d > 0) & (a > 0), a + tab_weight * d + 16, 0) + send_weight * d)
                               .astype(np.int64))

    # -- count --
    def _rows(self, sh):
        ip, ix = self._np(sh.indptr), self._np(sh.indices)
        return [ix[ip[v]: ip[v + 1]] for v in range(len(ip) - 1)]

    def _tab(self, sh, u):
        ip, ix = self._np(sh.indptr), self._np(sh.indices)
        return set(ix[ip[u - sh.lo]: ip[u - sh.lo + 1]].tolist())

    def _count_rows(self, sh, rows):
        c = 0
        for x in rows:
            for i, u in enumerate(x.tolist()):
                if sh.lo <= u < sh.hi and i + 1 < len(x):
                    c += len(set(x[i + 1:].tolist()) & self._tab(sh, u))
        return c

    def start_local(self, sh):
        return torch.tensor([self._count_rows(sh, self._rows(sh))]), None

    def send_sizes(self, sh, P, rank):
        b = np.asarray(sh.bounds, np.int64)
        out = np.zeros((3, P), np.int64)
        for x in self._rows(sh):
            d = len(x)
            for j in range(rank + 1, P):
                s, e = np.searchsorted(x, b[j]), np.searchsorted(x, b[j + 1])
                if s < e:  # the message starts at the 16-byte chunk of the first id >= b[j]
                    out[0, j] += 1
                    out[1, j] += ((d + 3) & ~3) - (s & ~3)
                    out[2, j] += d
        return None, out

    def send_pack(self, sh, P, rank, sizes_dev, nl, nw):
        b = np.asarray(sh.bounds, np.int64)
        lens, ids = [[] for _ in range(P)], [[] for _ in range(P)]
        for x in self._rows(sh):
            d = len(x)
            for j in range(rank + 1, P):
                s, e = np.searchsorted(x, b[j]), np.searchsorted(x, b[j + 1])
                if s < e:
                    s4 = s & ~3
                    lens[j].append(d - s4)
                    pl = ((d + 3) & ~3) - s4
                    ids[j].extend(x[s4:].tolist() + [self.IMAX] * (pl - (d - s4)))
        L = [v for j in range(P) for v in lens[j]]
        W = [v for j in range(P) for v in ids[j]]
        return torch.tensor(L, dtype=torch.int32), torch.tensor(W, dtype=torch.int32)

    def recv_pool(self, nw):
        buf = torch.full((self.HEAD + nw + 4,), self.IMAX, dtype=torch.int32)
        return buf, buf[self.HEAD: self.HEAD + nw]

    def count_received(self, sh, row_len, pool, key=None):
        p = self._np(pool)
        rows, off = [], 0
        for d in self._np(row_len).tolist():
            rows.append(p[off: off + d])
            off += (d + 3) & ~3
        return torch.tensor([self._count_rows(sh, rows)]), None

    def finish(self, outs):
        return int(sum(int(o.item()) for o in outs))
