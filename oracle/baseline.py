"""Timed CPU baseline of one composed training epoch -- TEST/BENCH INFRASTRUCTURE.

Used only by bench.py (the `cpu_baseline` object and `--impl reference`).
It runs the reference's CPU algorithm (numpy reduceat CSR aggregation,
kernels.py:87-134, row-chunked over a thread pool like kernels.py:126-131;
BLAS matmuls for the update, models.py:99) on a BOUNDED SAMPLE of the epoch:
every aggregation and GEMM of the epoch is run for the first R destination
rows only (the gathers still read the full-size feature matrices), and the
measured time is scaled by V / R.  The sample is reported with the number.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import time

import numpy as np


def _rows_csr(row_ptr, R_):
    """Sub-CSR of destination rows [0, R_)."""
    e = int(row_ptr[R_])
    return row_ptr[:R_ + 1].copy(), e


def _agg_rows(row_ptr, col, val, x, R_, threads):
    rp, e = _rows_csr(row_ptr, R_)
    out = np.empty((R_, x.shape[1]), np.float32)
    bounds = np.linspace(0, R_, threads + 1).astype(np.int64)

    def work(k):
        a, b = int(bounds[k]), int(bounds[k + 1])
        if a == b:
            return
        sub = (rp[a:b + 1] - rp[a]).astype(np.int32)
        e0, e1 = int(rp[a]), int(rp[b])
        out[a:b] = _reduce(sub, col[e0:e1], None if val is None else val[e0:e1], x, b - a)

    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(work, range(threads)))
    return out


def _reduce(rp, col, val, x, nrows):
    """np.add.reduceat over fl(val * x[col]) for non-empty rows (kernels.py:112-113)."""
    out = np.zeros((nrows, x.shape[1]), np.float32)
    counts = np.diff(rp)
    nz = np.flatnonzero(counts)
    if nz.size:
        starts = rp[:-1][nz].astype(np.int64)
        contrib = x[col] if val is None else val[:, None] * x[col]
        out[nz] = np.add.reduceat(contrib, starts, axis=0)
    return out


def epoch_sample(V, fwd, bwd, dims, rows: int, threads: int | None = None, seed: int = 0):
    """Time the sampled epoch.  fwd/bwd = (row_ptr, col, val|None) host CSR of
    A_hat and A_hat^T.  Returns (extrapolated epoch ms, sample description)."""
    threads = threads or os.cpu_count() or 1
    rows = min(rows, V)
    rng = np.random.default_rng(seed)
    fmax = max(dims[:-1])
    xs = rng.standard_normal((V, fmax), dtype=np.float32)
    ws = [rng.uniform(-0.1, 0.1, (dims[i], dims[i + 1])).astype(np.float32)
          for i in range(len(dims) - 1)]
    L = len(dims) - 1
    t0 = time.perf_counter()
    aggs = []
    for l in range(L):
        x = np.ascontiguousarray(xs[:, :dims[l]])
        agg = _agg_rows(*fwd, x, rows, threads)
        out = agg @ ws[l]
        if l < L - 1:
            np.maximum(out, 0, out=out)
        aggs.append(agg)
    g = rng.standard_normal((rows, dims[-1])).astype(np.float32)
    for l in range(L - 1, -1, -1):
        _ = aggs[l].T @ g
        if l == 0:
            break
        d_in = g @ ws[l].T
        full = np.ascontiguousarray(xs[:, :dims[l]])
        full[:rows] = d_in
        g = _agg_rows(*bwd, full, rows, threads)
    elapsed = time.perf_counter() - t0
    ms = elapsed * 1000.0 * V / rows
    sample = (f"first {rows} of {V} destination rows of every aggregation and GEMM of one "
              f"epoch (dims {dims}), scaled by V/rows; {threads} threads; measured {elapsed:.2f} s")
    return ms, sample
