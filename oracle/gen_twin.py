"""TEST INFRASTRUCTURE: numpy twin of the device generators (csrc/gen.cu).

The product generates configs 1/3/4/5 on the device (csrc/gen.cu).  This
module is the bit-identical numpy twin used to (a) produce golden fixtures
in this GPU-less container and (b) document the exact streams.  It is pure
integer arithmetic, mod 2**64.

    mix(z)       = splitmix64 finaliser (same constants as the reference's
                   pa_edge_list, _kernels.py:159-161)
    key(seed,s)  = mix(seed * 0xD1B54A32D192ED03 + s)       (stream key)
    rnd(key, i)  = mix(key + (i + 1) * 0x9E3779B97F4A7C15)  (i-th draw)
    mulhi(r, n)  = floor(r * n / 2**64)                       (n < 2**32)
"""

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
SEEDMUL = np.uint64(0xD1B54A32D192ED03)
MASK32 = np.uint64(0xFFFFFFFF)

STREAM_ER = 1
STREAM_RMAT = 2
STREAM_CL = 3

# R-MAT quadrant thresholds (a, a+b, a+b+c) = (0.57, 0.76, 0.95) as 2**64 fractions
RMAT_T = [int(0.57 * 2**64), int(0.76 * 2**64), int(0.95 * 2**64)]


def mix(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def key(seed, stream):
    with np.errstate(over="ignore"):
        return mix(np.uint64(seed) * SEEDMUL + np.uint64(stream))


def rnd(k, i):
    i = np.asarray(i, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix(np.uint64(k) + (i + np.uint64(1)) * GAMMA)


def mulhi(r, n):
    r = np.asarray(r, dtype=np.uint64)
    n = np.uint64(n)
    with np.errstate(over="ignore"):
        hi = (r >> np.uint64(32)) * n + (((r & MASK32) * n) >> np.uint64(32))
    return hi >> np.uint64(32)


def er_gnm(n, m, seed):
    """Config 1/5 raw pairs: m ordered pairs i.i.d. uniform on [0,n)^2
    (self-loops and duplicates kept; normalize() removes them)."""
    k = key(seed, STREAM_ER)
    i = np.arange(m, dtype=np.uint64)
    u = mulhi(rnd(k, 2 * i), n)
    v = mulhi(rnd(k, 2 * i + np.uint64(1)), n)
    return np.stack([u, v], axis=1).astype(np.int32)


def rmat(scale, edge_factor, seed):
    """Config 4 raw pairs: 2**scale * edge_factor samples, one draw per level
    choosing a quadrant against (0.57, 0.76, 0.95); no vertex permutation."""
    k = key(seed, STREAM_RMAT)
    ns = (1 << scale) * edge_factor
    i = np.arange(ns, dtype=np.uint64)
    src = np.zeros(ns, np.uint64)
    dst = np.zeros(ns, np.uint64)
    t0, t1, t2 = (np.uint64(t) for t in RMAT_T)
    for lvl in range(scale):
        r = rnd(k, i * np.uint64(scale) + np.uint64(lvl))
        bit = np.uint64(scale - 1 - lvl)
        sb = (r >= t1).astype(np.uint64)
        db = (((r >= t0) & (r < t1)) | (r >= t2)).astype(np.uint64)
        src |= sb << bit
        dst |= db << bit
    return np.stack([src, dst], axis=1).astype(np.int32)


def checksum(a):
    """Order-sensitive 64-bit checksum used by fixtures: sum((a+1)*(2i+1)) mod 2**64."""
    a = np.ascontiguousarray(np.asarray(a).ravel()).astype(np.int64).astype(np.uint64)
    w = np.arange(len(a), dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    with np.errstate(over="ignore"):
        return int(np.sum((a + np.uint64(1)) * w, dtype=np.uint64))
