"""numpy restatement of the reference AdaptGear path -- TEST INFRASTRUCTURE ONLY.

Each function cites the reference code it restates (paths relative to
/root/reference/pkg/src/adaptgear/).  Arrays are plain numpy; graphs are
(V, dst, src, w) with w None for unweighted graphs.  Pinned against the
golden vectors of tests/golden/ by tests/test_oracle.py.
"""
from __future__ import annotations

import heapq

import numpy as np

F32 = np.float32


# ------------------------------------------------------------------ graphs --
def canonical(V, dst, src, w=None):
    """Graph.from_edges (graph.py:47-82): sort by dst*V+src, dedup, fp64 merge."""
    d = np.asarray(dst, dtype=np.int64)
    s = np.asarray(src, dtype=np.int64)
    key = d * V + s
    uniq, inv = np.unique(key, return_inverse=True)
    wo = None
    if w is not None:
        # fp64 sum of duplicates in input order: np.bincount accumulates
        # sequentially like np.add.at (the reference's merge), bit for bit
        acc = np.bincount(inv.ravel(), weights=np.asarray(w, dtype=F32).astype(np.float64),
                          minlength=uniq.size)
        wo = acc.astype(F32)
    base = max(V, 1)
    return (uniq // base).astype(np.int32), (uniq % base).astype(np.int32), wo


def in_degrees(V, dst):
    """graph.py:94-96."""
    return np.bincount(np.asarray(dst), minlength=V).astype(np.int64)


def gcn_normalize(V, dst, src):
    """models.py:57-73: binary A+I, in-degree of A+I, w = f32(1/sqrt(d_i d_j)) in fp64."""
    loops = np.arange(V, dtype=np.int64)
    key = np.unique(np.concatenate([np.asarray(dst, np.int64) * V + np.asarray(src, np.int64),
                                    loops * V + loops]))
    d, s = key // V, key % V
    deg = np.bincount(d, minlength=V).astype(np.float64)
    w = (1.0 / np.sqrt(deg[d] * deg[s])).astype(F32)
    return canonical(V, d, s, w)


def apply_reorder(V, dst, src, w, perm):
    """reorder.py:217-228."""
    perm = np.asarray(perm, dtype=np.int64)
    return canonical(V, perm[np.asarray(dst)], perm[np.asarray(src)], w)


def decompose(V, dst, src, w, B):
    """decompose.py:57-75: intra iff floor(d/B) == floor(s/B); order preserved."""
    d = np.asarray(dst, np.int64)
    s = np.asarray(src, np.int64)
    m = (d // B) == (s // B)
    pick = (lambda a, k: None if a is None else a[k])
    intra = canonical(V, d[m], s[m], pick(w, m))
    inter = canonical(V, d[~m], s[~m], pick(w, ~m))
    return intra, inter, in_degrees(V, d)


# ----------------------------------------------------------------- formats --
def to_csr(V, dst, src, w):
    """formats.py:76-88."""
    row_ptr = np.zeros(V + 1, dtype=np.int32)
    np.cumsum(np.bincount(np.asarray(dst), minlength=V), out=row_ptr[1:])
    val = np.ones(len(dst), F32) if w is None else np.asarray(w, F32)
    return row_ptr, np.asarray(src, np.int32), val


def to_blocks(V, dst, src, w, B):
    """formats.py:105-140: stored communities, zero-padded B x B blocks, row_touched."""
    d = np.asarray(dst, np.int64)
    s = np.asarray(src, np.int64)
    c = d // B
    if np.any(c != s // B):
        raise ValueError("off-diagonal edge")
    ids = np.unique(c)
    blocks = np.zeros((ids.size, B, B), F32)
    touched = np.zeros((ids.size, B), bool)
    if ids.size:
        slot = np.searchsorted(ids, c)
        blocks[slot, d - c * B, s - c * B] = np.ones(d.size, F32) if w is None else w
        touched[slot, d - c * B] = True
    return ids.astype(np.int32), blocks, touched


# ----------------------------------------------------------------- kernels --
def csr_aggregate(V, row_ptr, col, val, x, op):
    """aggregate_csr_inter (kernels.py:87-134): np.add.reduceat over fl(val*x[col])
    per non-empty row (numpy's first-term + pairwise order); max over raw rows."""
    x = np.ascontiguousarray(x, dtype=F32)
    counts = np.diff(row_ptr)
    out = np.zeros((V, x.shape[1]), F32)
    nz = np.flatnonzero(counts)
    if nz.size:
        starts = row_ptr[:-1][nz].astype(np.int64)
        e1 = int(row_ptr[nz[-1] + 1])
        e0 = int(starts[0])
        cols = col[e0:e1]
        rel = starts - e0
        if op == "max":
            out[nz] = np.maximum.reduceat(x[cols], rel, axis=0)
        else:
            out[nz] = np.add.reduceat(val[e0:e1, None] * x[cols], rel, axis=0)
    return out, counts > 0


def coo_aggregate(V, row, col, val, x, op, chunk=1 << 19):
    """aggregate_coo_atomic (kernels.py:192-225): scrambled order, fp64 per chunk."""
    x = np.ascontiguousarray(x, dtype=F32)
    E = len(row)
    out = np.zeros((V, x.shape[1]), F32)
    touched = np.zeros(V, bool)
    if E == 0:
        return out, touched
    p = np.random.default_rng(E).permutation(E)
    r = np.asarray(row, np.int64)[p]
    c = np.asarray(col, np.int64)[p]
    v = np.asarray(val, F32)[p]
    touched[r] = True
    if op == "max":
        tmp = np.full(out.shape, -np.inf, F32)
        np.maximum.at(tmp, r, x[c])
        out[touched] = tmp[touched]
        return out, touched
    for k in range(0, E, chunk):
        rr = r[k:k + chunk]
        contrib = v[k:k + chunk, None] * x[c[k:k + chunk]]
        for j in range(x.shape[1]):
            out[:, j] += np.bincount(rr, weights=contrib[:, j], minlength=V).astype(F32)
    return out, touched


def dense_block_aggregate(V, B, ids, blocks, row_touched, x):
    """aggregate_dense_block (kernels.py:228-250)."""
    x = np.ascontiguousarray(x, dtype=F32)
    out = np.zeros((V, x.shape[1]), F32)
    touched = np.zeros(V, bool)
    if len(ids):
        idx = np.asarray(ids, np.int64)[:, None] * B + np.arange(B)[None, :]
        ok = idx < V
        xs = np.zeros((len(ids), B, x.shape[1]), F32)
        xs[ok] = x[idx[ok]]
        res = np.matmul(blocks, xs)
        out[idx[ok]] = res[ok]
        touched[idx[ok]] = row_touched[ok]
    return out, touched


def combine(a, ta, b, tb, op, deg=None):
    """combine (kernels.py:253-276)."""
    if op == "sum":
        return a + b
    if op == "mean":
        return (a + b) / np.maximum(np.asarray(deg), 1).astype(F32)[:, None]
    out = np.zeros_like(a)
    out[ta & ~tb] = a[ta & ~tb]
    out[tb & ~ta] = b[tb & ~ta]
    both = ta & tb
    out[both] = np.maximum(a[both], b[both])
    return out


def aggregate_full(V, dst, src, w, x, op):
    """aggregate_full (kernels.py:355-362): CSR + combine with an empty partial."""
    rp, col, val = to_csr(V, dst, src, w)
    vals, t = csr_aggregate(V, rp, col, val, x, op)
    z = np.zeros_like(vals)
    return combine(vals, t, z, np.zeros(V, bool), op, in_degrees(V, dst))


def aggregate_decomposed_csr(V, intra, inter, deg, x, op):
    """Decomposed aggregation with CSR kernels on both roles (bitwise target of
    the device csr_intra_blocked + csr_inter pair)."""
    a, ta = csr_aggregate(V, *to_csr(V, *intra), x, op)
    b, tb = csr_aggregate(V, *to_csr(V, *inter), x, op)
    return combine(a, ta, b, tb, op, deg)


def dense_reference(V, dst, src, w, x, op):
    """aggregate_dense_reference (kernels.py:286-306)."""
    x = np.ascontiguousarray(x, dtype=F32)
    if op == "max":
        rp, col, _ = to_csr(V, dst, src, w)
        vals, _ = csr_aggregate(V, rp, col, np.ones(len(col), F32), x, "max")
        return vals
    a = np.zeros((V, V), F32)
    a[np.asarray(dst), np.asarray(src)] = np.ones(len(dst), F32) if w is None else w
    out = a @ x
    if op == "mean":
        out = out / np.maximum(in_degrees(V, dst), 1).astype(F32)[:, None]
    return out.astype(F32)


def rel_error(values, reference) -> float:
    """conftest.py:22-26: max |a - ref| / max(|ref|, 1), in fp64."""
    ref = np.asarray(reference, dtype=np.float64)
    diff = np.abs(np.asarray(values, dtype=np.float64) - ref)
    return float((diff / np.maximum(np.abs(ref), 1.0)).max()) if diff.size else 0.0


# ----------------------------------------------------------------- reorder --
def _adjacency(V, dst, src):
    """reorder.py:44-53."""
    nb = [set() for _ in range(V)]
    for d, s in zip(np.asarray(dst).tolist(), np.asarray(src).tolist()):
        nb[d].add(s)
        nb[s].add(d)
    return [sorted(n) for n in nb]


def cluster_bfs(V, dst, src, B):
    """cluster_bfs (reorder.py:92-153) restated from SURVEY Appendix A.2."""
    adj = _adjacency(V, dst, src)
    deg = [len(a) for a in adj]
    seed_order = sorted(range(V), key=lambda v: (-deg[v], v))
    comm_of = [-1] * V
    placed = pos = comm = 0
    while placed < V:
        while comm_of[seed_order[pos]] >= 0:
            pos += 1
        start = seed_order[pos]
        comm_of[start] = comm
        placed += 1
        size = 1
        attach = {}
        heap = []
        for u in adj[start]:
            if comm_of[u] < 0:
                attach[u] = 1
                heapq.heappush(heap, (-1, u))
        while size < B and heap:
            neg, v = heapq.heappop(heap)
            if comm_of[v] >= 0 or attach.get(v, 0) != -neg:
                continue
            comm_of[v] = comm
            placed += 1
            size += 1
            del attach[v]
            for u in adj[v]:
                if comm_of[u] < 0:
                    attach[u] = attach.get(u, 0) + 1
                    heapq.heappush(heap, (-attach[u], u))
        comm += 1
    # _refine_swaps (reorder.py:56-89), 3 sweeps, Gauss-Seidel in id order
    members = {}
    for v, c in enumerate(comm_of):
        members.setdefault(c, []).append(v)
    for _ in range(3):
        moved = 0
        for v in range(V):
            if not adj[v]:
                continue
            c0 = comm_of[v]
            cnt = {}
            for u in adj[v]:
                cnt[comm_of[u]] = cnt.get(comm_of[u], 0) + 1
            cstar = min(cnt, key=lambda c: (-cnt[c], c))
            if cstar == c0 or cnt[cstar] <= cnt.get(c0, 0):
                continue
            best, best_u = 0, -1
            nv = set(adj[v])
            for u in sorted(members[cstar]):
                cu0 = sum(1 for t in adj[u] if comm_of[t] == c0)
                cus = sum(1 for t in adj[u] if comm_of[t] == cstar)
                delta = cnt[cstar] + cu0 - cnt.get(c0, 0) - cus - (2 if u in nv else 0)
                if delta > best:
                    best, best_u = delta, u
            if best_u >= 0:
                comm_of[v], comm_of[best_u] = cstar, c0
                members[c0].remove(v)
                members[cstar].append(v)
                members[cstar].remove(best_u)
                members[c0].append(best_u)
                moved += 1
        if not moved:
            break
    comm_arr = np.array(comm_of, dtype=np.int64)
    order = np.lexsort((np.arange(V), comm_arr))
    perm = np.empty(V, np.int64)
    perm[order] = np.arange(V)
    return comm_arr, perm


def partition_from_ids(ids, B):
    """load_partition core (reorder.py:177-203)."""
    ids = np.asarray(ids, np.int64)
    n = ids.size
    order = np.argsort(ids, kind="stable")
    comm = np.empty(n, np.int64)
    perm = np.empty(n, np.int64)
    chunk, within, prev = -1, 0, None
    for i, v in enumerate(order.tolist()):
        within = 0 if ids[v] != prev else within + 1
        prev = ids[v]
        if within % B == 0:
            chunk += 1
        comm[v] = chunk
        perm[v] = i
    return comm, perm


# ----------------------------------------------- composed training oracle --
def gnn_step(model, adj_fwd, adj_bwd, x, weights, labels, mask, gin_eps=0.0):
    """One composed GCN/GIN training step, fp32 numpy.

    adj_fwd / adj_bwd: callables F32[V,F] -> F32[V,F] applying A_hat (resp.
    A_hat^T) with the reference's aggregation.  Returns (loss, grads, logits).
    """
    s = F32(1.0 + gin_eps)
    L = len(weights)
    saved = []
    h = x.astype(F32)
    for l in range(L):
        agg = adj_fwd(h)
        if model == "gin":
            agg = s * h + agg
        out = (agg @ weights[l]).astype(F32)
        if l < L - 1:
            out = np.maximum(out, 0).astype(F32)
        saved.append((agg, out))
        h = out
    z = h.astype(np.float64)
    z = z - z.max(axis=1, keepdims=True)
    p = np.exp(z) / np.exp(z).sum(axis=1, keepdims=True)
    n = int(mask.sum())
    rows = np.flatnonzero(mask)
    loss = float(-np.log(p[rows, labels[rows]]).sum() / n)
    g = p.copy()
    g[rows, labels[rows]] -= 1.0
    g[~mask] = 0.0
    g = (g / n).astype(F32)
    grads = [None] * L
    for l in range(L - 1, -1, -1):
        agg, _ = saved[l]
        grads[l] = (agg.T @ g).astype(F32)
        if l == 0:
            break
        d_in = (g @ weights[l].T).astype(F32)
        d_h = adj_bwd(d_in)
        if model == "gin":
            d_h = s * d_in + d_h
        d_h = np.where(saved[l - 1][1] > 0, d_h, 0).astype(F32)
        g = d_h
    return loss, grads, h
