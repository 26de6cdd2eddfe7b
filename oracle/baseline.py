"""Timed CPU baseline of the composed training epoch -- TEST/BENCH INFRASTRUCTURE.

Used only by bench.py (the `cpu_baseline` object and `--impl reference`).  It
times the reference's own CPU kernels (numpy, as in pkg/src/adaptgear):

  forward, per layer, in the GPU path's association (a narrowing layer runs its
  update GEMM first, models.GNN.gemm_first): the intra role with the kernel the
  reference's selector locks on this host among csr_intra_blocked
  (kernels.py:137-189) and dense_block (kernels.py:228-250) -- timed on the
  first step, argmin as selector.py:120-154 -- the inter role with csr_inter
  (kernels.py:117-134), combine (kernels.py:253-276), the GIN (1+eps) x term
  (models.py:109-112), `agg @ W` (models.py:99, BLAS) and the ReLU;
  loss: mean masked softmax cross-entropy;
  backward: dW = agg^T G, d_in = G W^T, backward_sum (kernels.py:309-313: the
  CSR kernel over the transposed graph) and the ReLU mask; SGD.

coo_atomic is not a CPU candidate: its per-feature-column fp64 bincount
allocates and adds a V-length vector per column per 2^19-edge chunk
(kernels.py:219-224), i.e. F * V * E / 2^19 element operations -- at C5
F = 256 that is ~5e13, hours where csr_inter takes minutes.

Sizes: with `frac` = 1 the epoch runs on every row (C1-C3).  Otherwise a
uniform random sample of `frac` of the 16-row blocks (all their rows, every
edge of those rows, the GEMM rows of those rows) is run and every measured
time is scaled by V / sampled rows: each timed operation's cost is linear in
the rows / edges / blocks it processes, and the blocks are drawn uniformly,
so the scaled sum is an unbiased estimate of the full epoch.  Gathers read
full-size [V, F] source matrices, so memory behaviour matches the full run.
scripts/cpu_fullscale.py times full C5 aggregations to validate the scaling.

The CSR kernel is the reference's: np.add.reduceat over fl(val * x[col]) per
non-empty row; the reference's thread pool (kernels.py:126-131) is kept, but
numpy's reduceat holds the GIL, so it runs at one core's speed whatever the
thread count (measured; reported as `cores`).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import time

import numpy as np

from . import ref_numpy as R

F32 = np.float32
_PIECE_EDGES = 1 << 19  # kernels.py:35 chunk


def _sub_csr(row_ptr, col, val, rows):
    """CSR restricted to `rows` (same per-row edge order)."""
    rp = np.asarray(row_ptr, np.int64)
    cnt = rp[rows + 1] - rp[rows]
    sub = np.zeros(rows.size + 1, np.int64)
    np.cumsum(cnt, out=sub[1:])
    idx = np.repeat(rp[rows] - sub[:-1], cnt) + np.arange(sub[-1])
    return sub, np.asarray(col, np.int32)[idx], np.asarray(val, F32)[idx]


def csr_rows(rp, col, val, x, pool, threads):
    """aggregate_csr_inter's arithmetic on a (sub-)CSR: reduceat per non-empty
    row, rows split over the thread pool, edges in 2^19 pieces at row
    boundaries."""
    n = rp.size - 1
    out = np.zeros((n, x.shape[1]), F32)
    nz = np.flatnonzero(np.diff(rp))
    chunks = [c for c in np.array_split(nz, threads) if c.size]

    def work(c):
        a, b = int(c[0]), int(c[-1]) + 1
        r = a
        while r < b:
            q = int(np.searchsorted(rp, rp[r] + _PIECE_EDGES, side="right")) - 1
            q = min(max(q, r + 1), b)
            e0, e1 = int(rp[r]), int(rp[q])
            if e1 > e0:
                cnt = np.diff(rp[r:q + 1])
                nzr = np.flatnonzero(cnt)
                starts = (rp[r:q][nzr] - e0).astype(np.int64)
                out[r + nzr] = np.add.reduceat(val[e0:e1, None] * x[col[e0:e1]], starts, axis=0)
            r = q

    list(pool.map(work, chunks))
    return out


def dense_blocks(blocks, xs):
    """aggregate_dense_block's arithmetic (kernels.py:247): batched matmul."""
    return np.matmul(blocks, xs)


class SampledEpoch:
    def __init__(self, V, dst, src, w, B, dims, model, gin_eps=0.0, frac=1.0, seed=0,
                 threads=None):
        self.V, self.B, self.dims, self.model = V, B, list(dims), model
        self.scale_gin = F32(1.0 + gin_eps)
        self.threads = threads or os.cpu_count() or 1
        self.pool = cf.ThreadPoolExecutor(max_workers=self.threads)
        w = np.ones(len(dst), F32) if w is None else np.asarray(w, F32)
        (di, si, wi), (de, se, we), _ = R.decompose(V, dst, src, w, B)
        nb = (V + B - 1) // B
        rng = np.random.default_rng(seed)
        k = nb if frac >= 1.0 else max(1, int(round(frac * nb)))
        blk = np.arange(nb) if k == nb else np.sort(rng.choice(nb, size=k, replace=False))
        rows = (blk[:, None] * B + np.arange(B)[None, :]).ravel()
        self.rows = rows[rows < V]
        self.blocks_ids = blk
        self.scale = V / self.rows.size
        self.frac = self.rows.size / V
        self.intra = _sub_csr(*R.to_csr(V, di, si, wi), self.rows)
        self.inter = _sub_csr(*R.to_csr(V, de, se, we), self.rows)
        td, ts, tw = R.canonical(V, src, dst, w)
        self.bwd = _sub_csr(*R.to_csr(V, td, ts, tw), self.rows)
        # dense intra blocks of the sampled communities (formats.py:105-140)
        ids, blocks, _ = R.to_blocks(V, di, si, wi, B)
        pos = np.searchsorted(ids, blk)
        have = (pos < ids.size) & (ids[np.minimum(pos, ids.size - 1)] == blk)
        self.blocks = np.zeros((blk.size, B, B), F32)
        self.blocks[have] = blocks[pos[have]]
        self.block_rows = (blk[:, None] * B + np.arange(B)[None, :])
        self.choice = {}
        self.sample_edges = int(self.intra[0][-1] + self.inter[0][-1])

    def close(self):
        self.pool.shutdown()

    def gemm_first(self, l):
        return self.dims[l + 1] < self.dims[l]

    def _intra(self, kind, x):
        if kind == "dense_block":
            br = self.block_rows
            ok = br < self.V
            xs = np.zeros((br.shape[0], self.B, x.shape[1]), F32)
            xs[ok] = x[br[ok]]
            res = dense_blocks(self.blocks, xs)
            return res.reshape(-1, x.shape[1])[ok.ravel()]
        return csr_rows(*self.intra, x, self.pool, self.threads)

    def aggregate(self, key, x, timing):
        """Sampled rows of A_hat x: intra (selector-locked kernel) + inter
        (csr_inter) + combine; key = (direction, width) for the lock."""
        if key not in self.choice:  # the selector's profiling: one timed run each
            best = None
            for kind in ("csr_intra_blocked", "dense_block"):
                t0 = time.perf_counter()
                self._intra(kind, x)
                dt = time.perf_counter() - t0
                if best is None or dt < best[1]:
                    best = (kind, dt)
            self.choice[key] = best[0]
        t0 = time.perf_counter()
        a = self._intra(self.choice[key], x)
        b = csr_rows(*self.inter, x, self.pool, self.threads)
        a += b  # combine(sum)
        if self.model == "gin":
            a = self.scale_gin * x[self.rows] + a
        timing["agg"] += time.perf_counter() - t0
        return a

    def step(self, srcs, weights, labels, mask):
        """One sampled epoch.  srcs[f] = full-size [V, f] source matrix (the
        gathers' operands).  Returns the per-part wall seconds (unscaled)."""
        tm = {"agg": 0.0, "gemm": 0.0, "bwd_agg": 0.0, "other": 0.0}
        L = len(weights)
        rows = self.rows
        saved = []
        h = srcs[self.dims[0]][rows]
        for l in range(L):
            last = l == L - 1
            f_in, f_out = self.dims[l], self.dims[l + 1]
            if self.gemm_first(l):
                t0 = time.perf_counter()
                _ = h @ weights[l]  # this layer's GEMM rows (P = H W)
                tm["gemm"] += time.perf_counter() - t0
                out = self.aggregate(("fwd", f_out), srcs[f_out], tm)
                saved.append(("gemm", h))
            else:
                agg = self.aggregate(("fwd", f_in), srcs[f_in], tm)
                t0 = time.perf_counter()
                out = agg @ weights[l]
                tm["gemm"] += time.perf_counter() - t0
                saved.append(("agg", agg))
            t0 = time.perf_counter()
            if not last:
                np.maximum(out, 0, out=out)
            tm["other"] += time.perf_counter() - t0
            saved[-1] = saved[-1] + (out,)
            h = out
        t0 = time.perf_counter()
        z = h.astype(np.float64)
        z -= z.max(axis=1, keepdims=True)
        p = np.exp(z)
        p /= p.sum(axis=1, keepdims=True)
        lab, m = labels[rows], mask[rows]
        sel = np.flatnonzero(m)
        n = max(int(mask.sum()), 1)
        p[sel, lab[sel]] -= 1.0
        p[~m] = 0.0
        g = (p / n).astype(F32)
        tm["other"] += time.perf_counter() - t0
        grads = [None] * L
        for l in range(L - 1, -1, -1):
            kind, operand, _ = saved[l]
            h_prev = saved[l - 1][2] if l > 0 else None
            if kind == "agg":
                t0 = time.perf_counter()
                grads[l] = operand.T @ g
                tm["gemm"] += time.perf_counter() - t0
                if l == 0:
                    break
                t0 = time.perf_counter()
                _ = g @ weights[l].T  # d_in rows
                tm["gemm"] += time.perf_counter() - t0
                t0 = time.perf_counter()
                dh = csr_rows(*self.bwd, srcs[self.dims[l]], self.pool, self.threads)
                tm["bwd_agg"] += time.perf_counter() - t0
            else:
                t0 = time.perf_counter()
                q = csr_rows(*self.bwd, srcs[self.dims[l + 1]], self.pool, self.threads)
                tm["bwd_agg"] += time.perf_counter() - t0
                t0 = time.perf_counter()
                grads[l] = operand.T @ q
                if l == 0:
                    tm["gemm"] += time.perf_counter() - t0
                    break
                dh = q @ weights[l].T
                tm["gemm"] += time.perf_counter() - t0
            t0 = time.perf_counter()
            dh[h_prev <= 0] = 0.0
            g = dh
            tm["other"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        for wt, dw in zip(weights, grads):
            wt -= F32(0.01) * dw
        tm["other"] += time.perf_counter() - t0
        return tm


def make_inputs(V, dims, seed=0):
    rng = np.random.default_rng(seed)
    srcs = {f: rng.standard_normal((V, f), dtype=np.float32) for f in sorted(set(dims[:-1]) |
                                                                              set(dims[1:]))}
    ws = [rng.uniform(-0.1, 0.1, (dims[i], dims[i + 1])).astype(F32)
          for i in range(len(dims) - 1)]
    labels = rng.integers(0, dims[-1], V)
    mask = rng.random(V) < 0.5
    return srcs, ws, labels, mask


def time_epochs(V, dst, src, w, B, dims, model, frac, reps, warmup=1, seed=0, threads=None,
                gin_eps=0.0, budget_s=None):
    """Scaled epoch ms over `reps` sampled epochs (median) after `warmup`
    (the first warm-up step is the selector's profiling).  Returns a dict."""
    ep = SampledEpoch(V, dst, src, w, B, dims, model, gin_eps=gin_eps, frac=frac, seed=seed,
                      threads=threads)
    srcs, ws, labels, mask = make_inputs(V, dims, seed)
    try:
        for _ in range(max(1, warmup)):
            ep.step(srcs, ws, labels, mask)
        runs = []
        t_all = time.perf_counter()
        for _ in range(reps):
            t0 = time.perf_counter()
            parts = ep.step(srcs, ws, labels, mask)
            runs.append((time.perf_counter() - t0, parts))
            if budget_s is not None and time.perf_counter() - t_all > budget_s:
                break
        runs.sort(key=lambda r: r[0])
        wall, parts = runs[len(runs) // 2]
        return {"epoch_ms": wall * ep.scale * 1e3, "sample_wall_s": wall, "reps": len(runs),
                "parts_ms": {k: round(v * ep.scale * 1e3, 1) for k, v in parts.items()},
                "frac_rows": ep.frac, "sample_rows": int(ep.rows.size),
                "sample_edges": ep.sample_edges, "threads": ep.threads,
                "intra_choice": {f"{d}:{f}": k for (d, f), k in ep.choice.items()}}
    finally:
        ep.close()
