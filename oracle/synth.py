"""numpy restatement of the seeded generator -- TEST INFRASTRUCTURE ONLY.

Mirrors paper_2305_17408_b200/csrc/ag_prep.cu synth_kernel / vertex_keys_kernel
and paper_2305_17408_b200/synth.py community_graph operation for operation
(uint64 wrap-around hashing, IEEE double products, floor), so the device
generator can be checked bit-for-bit at small sizes.
"""
from __future__ import annotations

import numpy as np

from . import ref_numpy

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _unit(h):
    return (h >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def _scaled(u, n):
    v = np.floor(u * np.asarray(n, dtype=np.float64)).astype(np.int64)
    return np.minimum(v, np.asarray(n, np.int64) - 1)


def candidates(V, Bg, p_intra, p_global, window, skew, seed, first, count):
    seedmix = mix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF))
    i = np.arange(first, first + count, dtype=np.uint64)
    h = [mix64(seedmix ^ (i * np.uint64(8) + np.uint64(k))) for k in range(6)]
    u = [_unit(x) for x in h]
    p = u[0].copy()
    for _ in range(1, skew):
        p = p * u[0]
    d = _scaled(p, V)
    c = d // Bg
    base = c * Bg
    sz = np.minimum(Bg, V - base)
    nb = (V + Bg - 1) // Bg
    intra = (u[1] < p_intra) & (sz > 1)
    tt = _scaled(u[2], np.maximum(sz - 1, 1))
    s_intra = base + tt + (tt >= d - base)
    glob = u[3] < p_global
    cs_g = _scaled(u[4], nb)
    off = 1 + _scaled(u[4], window)
    sgn = np.where((h[5] & np.uint64(1)) == 1, 1, -1)
    cs_l = ((c + sgn * off) % nb + nb) % nb
    cs = np.where(glob, cs_g, cs_l)
    bs = cs * Bg
    szs = np.minimum(Bg, V - bs)
    s_inter = bs + _scaled(u[2], szs)
    s_inter = np.where(s_inter == d, -1, s_inter)
    s = np.where(intra, s_intra, s_inter)
    d = np.where(s < 0, -1, d)
    return d, s


def vertex_permutation(V, seed):
    keys = mix64(mix64(np.uint64((seed ^ 0xA5A5A5A5A5A5A5A5) & 0xFFFFFFFFFFFFFFFF))
                 ^ np.arange(V, dtype=np.uint64))
    order = np.argsort(keys, kind="stable")
    perm = np.empty(V, np.int64)
    perm[order] = np.arange(V)
    return perm


def _candidates_threaded(V, Bg, p_intra, p_global, window, skew, seed, n, threads=None):
    """candidates(..., 0, n) computed in index chunks on a thread pool (numpy
    releases the GIL in its ufuncs); candidate i depends on i alone, so the
    result is identical to one call."""
    import concurrent.futures as cf
    import os
    threads = threads or os.cpu_count() or 1
    if n < (1 << 20) or threads == 1:
        return candidates(V, Bg, p_intra, p_global, window, skew, seed, 0, n)
    step = (n + threads - 1) // threads
    parts = [(a, min(n, a + step)) for a in range(0, n, step)]
    d = np.empty(n, np.int64)
    s = np.empty(n, np.int64)

    def work(ab):
        a, b = ab
        d[a:b], s[a:b] = candidates(V, Bg, p_intra, p_global, window, skew, seed, a, b - a)

    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(work, parts))
    return d, s


def community_graph(V, E, block_gen=16, p_intra=0.5, p_global=0.1, window=4, skew=1, seed=0):
    n = E + E // 16 + 1024
    while True:
        d, s = _candidates_threaded(V, block_gen, p_intra, p_global, window, skew, seed, n)
        ok = s >= 0
        keys = d[ok] * V + s[ok]
        idx = np.arange(n, dtype=np.int64)[ok]
        uniq, first_pos = np.unique(keys, return_index=True)
        if uniq.size >= E:
            break
        n += 2 * (E - uniq.size) + 1024
    first = idx[first_pos]
    chosen = uniq[np.argsort(first, kind="stable")[:E]]
    perm = vertex_permutation(V, seed)
    dst, src, _ = ref_numpy.canonical(V, perm[chosen // V], perm[chosen % V])
    comm = np.empty(V, np.int64)
    comm[perm] = np.arange(V) // block_gen
    return (dst, src), comm
