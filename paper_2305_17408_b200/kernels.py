"""Density-specialised aggregation kernels (reference kernels.py:31-376).

Same operator API as the reference; every kernel is a hand-written sm_100a
kernel behind the C ABI:

  csr_inter          ag_fused_spmm          slab kernel (TMA-fed smem X ring), values
                                            bitwise equal to the reference's
                                            np.add.reduceat order
  csr_intra_blocked  ag_csr_intra_spmm      per-community smem-staged slab (the
                                            public call, honouring the tile
                                            budget); ag_fused_spmm inside the
                                            decomposed runtime (same bits)
  coo_atomic         ag_coo_spmm            edge-parallel, vector atomics
  dense_block        ag_dense_block_spmm    batched B x B block products
  dense_reference    dense adjacency @ X on the device (ag_gemm_f32), V <= cap

The decomposed path with a CSR x CSR pair is ONE launch of ag_fused_spmm over
the full reordered CSR: both role sums in the reference's order and
combine() in the epilogue, one output write.  Other pairs run the inter role
first (raw partial, or atomics into a zero / -inf buffer) and the intra role
second with combine() fused into its epilogue (AG_EPI_COMBINE).  Outputs are fresh CUDA tensors; `threads` is accepted for
signature compatibility and ignored.
"""
from __future__ import annotations

import enum
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .decompose import DecomposedGraph, full_graph
from .errors import KernelError
from .formats import CooMatrix, CsrMatrix, DenseBlockSet, to_coo, to_csr, to_dense_blocks
from .graph import Graph, as_device

DEFAULT_TILE_BUDGET_BYTES = 48 * 1024
DENSE_ORACLE_CAP = 4096
PRESPLIT_MAX_ELEMS = 1 << 20  # B operands up to 4 MB get a precomputed tf32 lo half


class AggregateOp(enum.Enum):
    SUM = "sum"
    MEAN = "mean"
    MAX = "max"


class KernelKind(enum.Enum):
    CSR_INTER = "csr_inter"
    CSR_INTRA_BLOCKED = "csr_intra_blocked"
    COO_ATOMIC = "coo_atomic"
    DENSE_BLOCK = "dense_block"
    DENSE_REFERENCE = "dense_reference"


@dataclass
class PartialResult:
    """One subgraph's aggregation before combination; untouched rows hold 0."""

    values: torch.Tensor
    touched: torch.Tensor
    op: AggregateOp
    note: str | None = None


def _opcode(op: AggregateOp) -> int:
    return _lib.AG_OP[op.value]


def _check_features(num_vertices: int, x) -> torch.Tensor:
    x = as_device(x, torch.float32)
    if x.dim() != 2 or x.shape[0] != num_vertices:
        raise KernelError(
            f"feature matrix shape {tuple(x.shape)} does not match {num_vertices} vertices")
    return x


def empty_partial(num_vertices: int, dim: int, op: AggregateOp) -> PartialResult:
    dev = _lib.device()
    return PartialResult(values=torch.zeros((num_vertices, dim), dtype=torch.float32, device=dev),
                         touched=torch.zeros(num_vertices, dtype=torch.bool, device=dev), op=op)


# ------------------------------------------------------------ raw launches --
def launch_csr(a: CsrMatrix, x: torch.Tensor, y: torch.Tensor, op: AggregateOp, flags: int = 0,
               other_touched: torch.Tensor | None = None, deg: torch.Tensor | None = None,
               gin_scale: float = 0.0) -> None:
    _lib.call("ag_csr_spmm", a.num_vertices, x.shape[1], _lib.ptr(a.row_ptr),
              _lib.ptr(a.col_idx), _lib.ptr(a.kernel_val), _lib.ptr(x), _lib.ptr(y),
              _opcode(op), flags, _lib.ptr(other_touched), _lib.ptr(deg), float(gin_scale),
              _lib.stream())


def relu_words(feat: int) -> int:
    """uint32 words per row of a bit-packed ReLU mask (include/adaptgear_b200.h)."""
    return (feat + 31) // 32


def relu_bits_empty(rows: int, feat: int, dev) -> torch.Tensor:
    """Uninitialised [rows, ceil(feat / 32)] int32 relu-bit mask (bit c % 32 of
    word c // 32 = activation > 0)."""
    return torch.empty((rows, relu_words(feat)), dtype=torch.int32, device=dev)


def relu_bits(h: torch.Tensor) -> torch.Tensor:
    """The relu-bit mask of an fp32 activation (ag_relu_bits)."""
    out = relu_bits_empty(h.shape[0], h.shape[1], h.device)
    _lib.call("ag_relu_bits", h.shape[0], h.shape[1], _lib.ptr(h), h.stride(0), _lib.ptr(out),
              out.stride(0), _lib.stream())
    return out


def _bits_for(relu_src, relu_bits_in, rows: int, feat: int):
    """A relu-bit mask for the kernels: given bits (checked) or built from an
    fp32 relu_src."""
    if relu_bits_in is not None:
        if relu_bits_in.dtype != torch.int32 or tuple(relu_bits_in.shape) != (rows, relu_words(feat)) \
                or not relu_bits_in.is_contiguous():
            raise ValueError(f"relu bits must be a contiguous int32 [{rows}, {relu_words(feat)}] mask")
        return relu_bits_in
    if relu_src is None:
        return None
    if tuple(relu_src.shape) != (rows, feat):
        raise ValueError(f"relu_src must have shape [{rows}, {feat}]")
    return relu_bits(relu_src)


_BAND_FLAGS = None
GATHER_MAX_BYTES = 64 << 20  # features up to this size take the gather pair (they stay in L2)
GATHER_MIN_COVERAGE = 0.9     # below this ring coverage the slab kernel's general path dominates


def _gather_ok(a: CsrMatrix, x: torch.Tensor, y: torch.Tensor, flags: int) -> bool:
    """The order-free (dense_block, coo_atomic) pair runs as one row gather
    (ag_gather_pair_spmm) when the features fit L2, or when the slab kernel's
    ring would serve under 90% of the edges (wide windows, many global
    edges: its general path's per-edge global loads cost more than a plain
    L2 gather).  AG_GATHER=0 disables it, AG_GATHER=2 forces it."""
    mode = os.environ.get("AG_GATHER", "1")
    if mode == "0":
        return False
    F = x.shape[1]
    allowed = (_lib.AG_EPI_GIN | _lib.AG_EPI_RELU | _lib.AG_EPI_RELU_MASK
               | _lib.AG_EPI_INTER_COO)
    if not (F % 4 == 0 and x.stride(0) == F and y.stride(0) == F and x.data_ptr() % 16 == 0
            and y.data_ptr() % 16 == 0 and (flags & ~allowed) == 0
            and x.shape[0] == a.num_vertices):
        return False
    return (mode == "2" or x.shape[0] * F * 4 <= GATHER_MAX_BYTES
            or a.ring_coverage() < GATHER_MIN_COVERAGE)


def _band_ok(x: torch.Tensor, y: torch.Tensor, rb, flags: int) -> bool:
    """The band kernel (ag_band_spmm) takes this order-free dense + coo launch:
    feat % 4 == 0 and > 32, 16-byte aligned operands, GIN / RELU / RELU_MASK
    epilogues only.  Opt-in (AG_BAND=1): measured slower than the slab
    kernel's dense + coo mode at every C5 width ("band kernel")."""
    global _BAND_FLAGS
    if _BAND_FLAGS is None:
        _BAND_FLAGS = (_lib.AG_EPI_GIN | _lib.AG_EPI_RELU | _lib.AG_EPI_RELU_MASK
                       | _lib.AG_EPI_INTER_COO)
    if os.environ.get("AG_BAND", "0") != "1":
        return False
    F = x.shape[1]
    return (F % 4 == 0 and F > 32 and x.stride(0) == F and y.stride(0) == F
            and x.data_ptr() % 16 == 0 and y.data_ptr() % 8 == 0
            and (rb is None or rb.data_ptr() % 16 == 0) and (flags & ~_BAND_FLAGS) == 0)


def launch_fused(a: CsrMatrix, x: torch.Tensor, y: torch.Tensor, op: AggregateOp,
                 block: int = 0, mask: int = 2, flags: int = 0,
                 other_touched: torch.Tensor | None = None, deg: torch.Tensor | None = None,
                 gin_scale: float = 0.0, relu_src: torch.Tensor | None = None,
                 dense_intra: bool = False, relu_bits_in: torch.Tensor | None = None,
                 relu_out: torch.Tensor | None = None) -> None:
    """ag_fused_spmm: slab (smem X ring) row gather, reduceat-order reduction (+ role split).

    block > 0 splits every row into its intra run and inter edges (role-ordered
    copy of the CSR, built once); block == 0 treats the row as one role.
    relu_src (fp32) / relu_bits_in (bit mask) apply the ReLU backward of the
    layer below in the epilogue; relu_out receives y's relu bits (with
    AG_EPI_RELU in flags).
    """
    rb = _bits_for(relu_src, relu_bits_in, a.num_vertices, x.shape[1])
    if relu_out is not None:
        _bits_for(None, relu_out, a.num_vertices, x.shape[1])
    if dense_intra and block == 16 and mask == 3 and op is AggregateOp.SUM \
            and (flags & _lib.AG_EPI_INTER_COO) and _gather_ok(a, x, y, flags):
        # a small graph: the order-free pair as one row gather (no ring start-up)
        _lib.call("ag_gather_pair_spmm", a.num_vertices, x.shape[1], _lib.ptr(a.row_ptr),
                  _lib.ptr(a.col_idx), _lib.ptr(a.kernel_val), _lib.ptr(x), _lib.ptr(y),
                  flags & ~_lib.AG_EPI_INTER_COO | (_lib.AG_EPI_RELU_MASK if rb is not None else 0),
                  float(gin_scale), _lib.ptr(rb), _lib.ptr(relu_out), _lib.stream())
        return
    if dense_intra and block == 16 and mask == 3 and op is AggregateOp.SUM \
            and (flags & _lib.AG_EPI_INTER_COO) and _band_ok(x, y, rb, flags):
        rec, off, far_cnt, far_src, window = a.band_layout()
        _lib.call("ag_band_spmm", a.num_vertices, x.shape[1], _lib.ptr(a.row_ptr), _lib.ptr(rec),
                  _lib.ptr(off), _lib.ptr(far_cnt), _lib.ptr(far_src), _lib.ptr(a.dense_blocks16()),
                  a.num_edges, _lib.ptr(x), _lib.ptr(y),
                  flags | (_lib.AG_EPI_RELU_MASK if rb is not None else 0), float(gin_scale),
                  _lib.ptr(rb), _lib.ptr(relu_out), x.shape[0], window, _lib.stream())
        return
    mid, cv, rowinfo, far_cnt, far_src, weighted = a.slab_layout(block)
    _lib.call("ag_fused_spmm", a.num_vertices, x.shape[1], int(mask), _lib.ptr(a.row_ptr),
              _lib.ptr(mid), _lib.ptr(cv), _lib.ptr(rowinfo), _lib.ptr(far_cnt),
              _lib.ptr(far_src), weighted,
              _lib.ptr(a.dense_blocks16() if dense_intra else None), a.num_edges, _lib.ptr(x), _lib.ptr(y),
              _opcode(op), flags | (_lib.AG_EPI_RELU_MASK if rb is not None else 0),
              _lib.ptr(other_touched), _lib.ptr(deg), float(gin_scale), _lib.ptr(rb),
              _lib.ptr(relu_out), x.shape[0], a.window(), _lib.stream())


def _check_block_local(a: CsrMatrix, block_size: int) -> None:
    bad = a.first_off_block(block_size)
    if bad >= 0:
        r = int(a.rows()[bad].item())
        c = int(a.col_idx[bad].item())
        raise KernelError(f"off-diagonal edge (dst={r}, src={c}) for block_size={block_size}")


def launch_csr_intra(a: CsrMatrix, x: torch.Tensor, y: torch.Tensor, op: AggregateOp,
                     block_size: int, tile_budget_bytes: int = DEFAULT_TILE_BUDGET_BYTES,
                     flags: int = 0, other_touched=None, deg=None, gin_scale: float = 0.0):
    if block_size < 1:
        raise KernelError("block_size must be >= 1")
    _check_block_local(a, block_size)
    _lib.call("ag_csr_intra_spmm", a.num_vertices, x.shape[1], int(block_size),
              int(tile_budget_bytes), _lib.ptr(a.row_ptr), _lib.ptr(a.col_idx),
              _lib.ptr(a.kernel_val), _lib.ptr(x), _lib.ptr(y), _opcode(op), flags,
              _lib.ptr(other_touched), _lib.ptr(deg), float(gin_scale), _lib.stream())


def launch_coo(a: CooMatrix, x: torch.Tensor, y: torch.Tensor, op: AggregateOp) -> None:
    """Accumulate into y (caller initialises 0 / -inf)."""
    _lib.call("ag_coo_spmm", a.num_vertices, x.shape[1], a.num_edges, _lib.ptr(a.row),
              _lib.ptr(a.col), _lib.ptr(a.kernel_val), _lib.ptr(x), _lib.ptr(y), _opcode(op),
              _lib.stream())


def coo_init(y: torch.Tensor, op: AggregateOp) -> None:
    y.fill_(float("-inf") if op is AggregateOp.MAX else 0.0)


def launch_dense_block(d: DenseBlockSet, x: torch.Tensor, y: torch.Tensor, op: AggregateOp,
                       flags: int = 0, other_touched=None, deg=None, gin_scale: float = 0.0):
    _lib.call("ag_dense_block_spmm", d.num_vertices, x.shape[1], d.block_size,
              _lib.ptr(d.comm_slot), _lib.ptr(d.blocks), _lib.ptr(d.row_touched), _lib.ptr(x),
              _lib.ptr(y), _opcode(op), flags, _lib.ptr(other_touched), _lib.ptr(deg),
              float(gin_scale), _lib.stream())


# dense_block on the tensor cores (tcgen05 3xTF32, fp32-faithful) from this
# block size up; below it the fp32 SIMT kernel (B = 16 blocks are HBM-bound and
# would need 8x the operand bytes as 128-wide panels).  SURVEY §2.2 K4.
DENSE_TC_MIN_BLOCK = 64


def dense_block_engine(d: DenseBlockSet, x: torch.Tensor, precision: str | None) -> str:
    """"tc" (ag_block_diag_gemm_tf32x3) or "simt" (ag_dense_block_spmm)."""
    if precision not in (None, "fp32", "tf32x3"):
        raise ValueError(f"unknown dense_block precision {precision!r}")
    tc_able = d.tc_ok() and _tc_ok(x) and x.shape[0] == d.num_vertices
    if precision == "tf32x3":
        if not tc_able:
            raise KernelError("tensor-core dense_block needs B dividing 128 or a multiple of 128 "
                              "and 16-byte aligned features with a row stride multiple of 4")
        return "tc"
    if precision is None and tc_able and d.block_size >= DENSE_TC_MIN_BLOCK:
        return "tc"
    return "simt"


def launch_dense_block_tc(d: DenseBlockSet, x: torch.Tensor, y: torch.Tensor,
                          beta: float = 0.0) -> None:
    """y = blockdiag(blocks) @ x (+ beta * y) on the tensor cores."""
    A = d.panels()
    _lib.call("ag_block_diag_gemm_tf32x3", d.num_vertices, x.shape[1], d.panel, _lib.ptr(A),
              A.stride(0), _lib.ptr(x), x.stride(0), x.shape[0], _lib.ptr(y), y.stride(0),
              float(beta), _lib.stream())


def _coo_touched(a: CooMatrix) -> torch.Tensor:
    t = torch.zeros(a.num_vertices, dtype=torch.bool, device=a.row.device)
    if a.num_edges:
        t[a.row.long()] = True
    return t


def _block_touched(d: DenseBlockSet) -> torch.Tensor:
    dev = d.blocks.device
    t = torch.zeros(d.num_vertices, dtype=torch.bool, device=dev)
    if d.community_ids.numel():
        idx = (d.community_ids.long()[:, None] * d.block_size
               + torch.arange(d.block_size, device=dev)[None, :])
        valid = idx < d.num_vertices
        t[idx[valid]] = d.row_touched[valid]
    return t


# -------------------------------------------------------------- public API --
def aggregate_csr_inter(a: CsrMatrix, x, op: AggregateOp, threads: int = 1) -> PartialResult:
    """Row-parallel CSR aggregation (the inter-subgraph kernel), kernels.py:117-134."""
    del threads
    x = _check_features(a.num_vertices, x)
    y = torch.empty((a.num_vertices, x.shape[1]), dtype=torch.float32, device=x.device)
    launch_fused(a, x, y, op)
    return PartialResult(values=y, touched=a.touched().clone(), op=op)


def aggregate_csr_intra_blocked(a: CsrMatrix, x, op: AggregateOp, block_size: int,
                                tile_budget_bytes: int = DEFAULT_TILE_BUDGET_BYTES,
                                threads: int = 1) -> PartialResult:
    """CSR aggregation with per-community smem staging, kernels.py:137-189.

    Bitwise identical to aggregate_csr_inter for any tile budget.
    """
    del threads
    if block_size < 1:
        raise KernelError("block_size must be >= 1")
    x = _check_features(a.num_vertices, x)
    y = torch.empty((a.num_vertices, x.shape[1]), dtype=torch.float32, device=x.device)
    launch_csr_intra(a, x, y, op, block_size, tile_budget_bytes)
    return PartialResult(values=y, touched=a.touched().clone(), op=op)


def aggregate_coo_atomic(a: CooMatrix, x, op: AggregateOp) -> PartialResult:
    """Edge-parallel aggregation with atomic accumulation, kernels.py:192-225.

    Sum / mean partials run as a row gather over the dst-sorted COO
    (ag_coo_gather_spmm: same order-free semantics, no atomics); max keeps the
    atomic compare-exchange kernel."""
    x = _check_features(a.num_vertices, x)
    y = torch.empty((a.num_vertices, x.shape[1]), dtype=torch.float32, device=x.device)
    if op is not AggregateOp.MAX and os.environ.get("AG_COO_ATOMIC") != "1":
        _lib.call("ag_coo_gather_spmm", a.num_vertices, x.shape[1], _lib.ptr(a.row_ptr),
                  _lib.ptr(a.col), _lib.ptr(a.kernel_val), _lib.ptr(x), _lib.ptr(y),
                  _lib.stream())
    else:
        coo_init(y, op)
        launch_coo(a, x, y, op)
    touched = _coo_touched(a)
    note = None
    if op is AggregateOp.MAX:
        note = "max via atomic compare-exchange emulation"
        y.masked_fill_(~touched[:, None], 0.0)
    return PartialResult(values=y, touched=touched, op=op, note=note)


def aggregate_dense_block(d: DenseBlockSet, x, op: AggregateOp,
                          precision: str | None = None) -> PartialResult:
    """Batched dense products over diagonal blocks, kernels.py:228-250 (no max).

    precision None picks the tensor cores (3xTF32) for B >= DENSE_TC_MIN_BLOCK
    and the fp32 SIMT kernel below; "fp32" / "tf32x3" force one.  The
    reference's BLAS matmul leaves the order unpinned (tolerance 1e-5)."""
    if op is AggregateOp.MAX:
        raise KernelError("dense_block kernel does not support max aggregation")
    x = _check_features(d.num_vertices, x)
    y = torch.empty((d.num_vertices, x.shape[1]), dtype=torch.float32, device=x.device)
    if dense_block_engine(d, x, precision) == "tc":
        launch_dense_block_tc(d, x, y)
    else:
        launch_dense_block(d, x, y, op)
    return PartialResult(values=y, touched=_block_touched(d), op=op)


def combine(intra: PartialResult, inter: PartialResult, op: AggregateOp,
            full_in_degree=None) -> torch.Tensor:
    """Merge intra and inter partial results, kernels.py:253-276."""
    if intra.op is not op or inter.op is not op:
        raise KernelError(f"op mismatch: combine({intra.op}, {inter.op}) as {op}")
    if intra.values.shape != inter.values.shape:
        raise KernelError("partial result shapes differ")
    deg = None
    if op is AggregateOp.MEAN:
        if full_in_degree is None:
            raise KernelError("mean combine requires the full-graph degree vector")
        deg = as_device(full_in_degree, torch.int64)
    a = as_device(intra.values, torch.float32)
    b = as_device(inter.values, torch.float32)
    ta = as_device(intra.touched, torch.bool) if op is AggregateOp.MAX else None
    tb = as_device(inter.touched, torch.bool) if op is AggregateOp.MAX else None
    out = torch.empty_like(a)
    _lib.call("ag_combine", a.shape[0], a.shape[1], _lib.ptr(a), _lib.ptr(ta), _lib.ptr(b),
              _lib.ptr(tb), _lib.ptr(deg), _opcode(op), _lib.ptr(out), _lib.stream())
    return out


def dense_adjacency(g: Graph) -> torch.Tensor:
    """V x V fp32 adjacency on the device."""
    a = torch.zeros((g.num_vertices, g.num_vertices), dtype=torch.float32, device=g.dst.device)
    if g.num_edges:
        a[g.dst.long(), g.src.long()] = g.edge_weights()
    return a


def _tc_ok(t: torch.Tensor) -> bool:
    return t.data_ptr() % 16 == 0 and t.stride(0) % 4 == 0 and t.stride(1) == 1


def gemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None, *,
         trans_a: bool = False, trans_b: bool = False, alpha: float = 1.0, beta: float = 0.0,
         relu: bool = False, relu_mask: torch.Tensor | None = None,
         engine: str = "auto", relu_mask_bits: torch.Tensor | None = None,
         mask_out: torch.Tensor | None = None) -> torch.Tensor:
    """out = alpha * op(a) @ op(b) + beta * out (the layers' update GEMM).

    engine "auto" runs the tcgen05 3xTF32 tensor-core kernel (ag_gemm_tf32x3)
    whenever the operands are 16-byte aligned with row strides that are
    multiples of 4 floats, else the fp32 SIMT kernel (ag_gemm_f32); "tc" /
    "simt" force one of them.  relu_mask fuses the ReLU backward of the layer
    below: out = relu_mask > 0 ? out : 0 (same shape as out); relu_mask_bits
    is the same as a bit-packed mask.  mask_out receives out's relu bits.
    """
    M = a.shape[1] if trans_a else a.shape[0]
    K = a.shape[0] if trans_a else a.shape[1]
    N = b.shape[0] if trans_b else b.shape[1]
    Kb = b.shape[1] if trans_b else b.shape[0]
    if K != Kb:
        raise KernelError(f"gemm inner dimensions differ: {K} vs {Kb}")
    if out is None:
        out = torch.empty((M, N), dtype=torch.float32, device=a.device)
    tc = engine == "tc" or (engine == "auto" and K > 0 and _tc_ok(a) and _tc_ok(b))
    epi = _lib.AG_GEMM_RELU if relu else 0
    mbits = _bits_for(relu_mask, relu_mask_bits, M, N)
    mask_ld = 0 if mbits is None else mbits.stride(0)
    if mask_out is not None:
        _bits_for(None, mask_out, M, N)
    mo_ld = 0 if mask_out is None else mask_out.stride(0)
    if tc:
        b_lo = None
        if b.shape[0] * b.stride(0) <= PRESPLIT_MAX_ELEMS:
            # a small B (the layer weights) is re-read by every output tile: split
            # its tf32 lo half once instead of in every tile's shared memory
            base = b.as_strided((b.shape[0], b.stride(0)), (b.stride(0), 1))
            b_lo = torch.empty_like(base)
            _lib.call("ag_tf32_split_lo", base.numel(), _lib.ptr(base), _lib.ptr(b_lo),
                      _lib.stream())
        _lib.call("ag_gemm_tf32x3", M, N, K, _lib.ptr(a), a.stride(0), int(trans_a), _lib.ptr(b),
                  b.stride(0), int(trans_b), _lib.ptr(b_lo), _lib.ptr(out), out.stride(0),
                  float(alpha), float(beta), epi, _lib.ptr(mbits), mask_ld, _lib.ptr(mask_out),
                  mo_ld, _lib.stream())
    else:
        _lib.call("ag_gemm_f32", M, N, K, _lib.ptr(a), a.stride(0), int(trans_a), _lib.ptr(b),
                  b.stride(0), int(trans_b), _lib.ptr(out), out.stride(0), float(alpha),
                  float(beta), epi, _lib.ptr(mbits), mask_ld, _lib.ptr(mask_out), mo_ld,
                  _lib.stream())
    return out


def aggregate_dense_reference(g: Graph, x, op: AggregateOp,
                              cap: int = DENSE_ORACLE_CAP) -> torch.Tensor:
    """Dense-adjacency aggregation on the device (kernels.py:286-306), V <= cap."""
    if g.num_vertices > cap:
        raise KernelError(f"dense oracle capped at {cap} vertices, got {g.num_vertices}")
    x = _check_features(g.num_vertices, x)
    if op is AggregateOp.MAX:
        y = torch.zeros((g.num_vertices, x.shape[1]), dtype=torch.float32, device=x.device)
        launch_csr(to_csr(g), x, y, op, flags=_lib.AG_EPI_COMBINE)
        return y
    out = gemm(dense_adjacency(g), x)
    if op is AggregateOp.MEAN:
        zeros = torch.zeros_like(out)
        _lib.call("ag_combine", out.shape[0], out.shape[1], _lib.ptr(out), None, _lib.ptr(zeros),
                  None, _lib.ptr(g.in_degrees()), _opcode(op), _lib.ptr(out), _lib.stream())
    return out


def backward_sum(g_transposed: Graph, d_y, threads: int = 1) -> torch.Tensor:
    """dX = A^T dY: sum-aggregation over the edge-reversed graph (kernels.py:309-313)."""
    return aggregate_csr_inter(to_csr(g_transposed), d_y, AggregateOp.SUM, threads).values


@dataclass
class SubgraphExec:
    """Pre-built device formats of one subgraph, reused across iterations."""

    graph: Graph
    block_size: int
    csr: CsrMatrix
    coo: CooMatrix
    blocks: DenseBlockSet | None = None

    @classmethod
    def for_intra(cls, g: Graph, block_size: int) -> "SubgraphExec":
        return cls(graph=g, block_size=block_size, csr=to_csr(g), coo=to_coo(g),
                   blocks=to_dense_blocks(g, block_size))

    @classmethod
    def for_inter(cls, g: Graph, block_size: int) -> "SubgraphExec":
        return cls(graph=g, block_size=block_size, csr=to_csr(g), coo=to_coo(g))

    def run(self, kind: KernelKind, x, op: AggregateOp,
            tile_budget_bytes: int = DEFAULT_TILE_BUDGET_BYTES, threads: int = 1) -> PartialResult:
        if kind is KernelKind.CSR_INTER:
            return aggregate_csr_inter(self.csr, x, op)
        if kind is KernelKind.CSR_INTRA_BLOCKED:
            return aggregate_csr_intra_blocked(self.csr, x, op, self.block_size,
                                               tile_budget_bytes=tile_budget_bytes)
        if kind is KernelKind.COO_ATOMIC:
            return aggregate_coo_atomic(self.coo, x, op)
        if kind is KernelKind.DENSE_BLOCK:
            if self.blocks is None:
                raise KernelError("dense_block kernel requires an intra subgraph")
            return aggregate_dense_block(self.blocks, x, op)
        if kind is KernelKind.DENSE_REFERENCE:
            values = aggregate_dense_reference(self.graph, x, op)
            return PartialResult(values=values, touched=self.csr.touched().clone(), op=op)
        raise KernelError(f"unknown kernel {kind}")

    # ---- fused two-role execution (used by the decomposed path) ----------
    def run_raw_into(self, kind: KernelKind, x: torch.Tensor, y: torch.Tensor,
                     op: AggregateOp, tile_budget_bytes: int) -> None:
        """First role: write this subgraph's raw partial into y.

        COO leaves untouched max rows at -inf; the second role's epilogue only
        reads y where this subgraph's `touched` is set.
        """
        if kind in (KernelKind.CSR_INTER, KernelKind.CSR_INTRA_BLOCKED):
            launch_fused(self.csr, x, y, op)
        elif kind is KernelKind.COO_ATOMIC:
            if op is not AggregateOp.MAX and os.environ.get("AG_COO_ATOMIC") != "1":
                _lib.call("ag_coo_gather_spmm", self.coo.num_vertices, x.shape[1],
                          _lib.ptr(self.coo.row_ptr), _lib.ptr(self.coo.col),
                          _lib.ptr(self.coo.kernel_val), _lib.ptr(x), _lib.ptr(y), _lib.stream())
            else:
                coo_init(y, op)
                launch_coo(self.coo, x, y, op)
        else:
            y.copy_(self.run(kind, x, op, tile_budget_bytes).values)

    def run_combine_into(self, kind: KernelKind, x: torch.Tensor, y: torch.Tensor,
                         op: AggregateOp, other_touched: torch.Tensor, deg: torch.Tensor,
                         tile_budget_bytes: int, gin_scale: float | None = None) -> None:
        """Second role: y = combine(this, y) [+ gin_scale * x], fused when possible."""
        flags = _lib.AG_EPI_COMBINE | (_lib.AG_EPI_GIN if gin_scale is not None else 0)
        g = 0.0 if gin_scale is None else gin_scale
        if kind in (KernelKind.CSR_INTRA_BLOCKED, KernelKind.CSR_INTER):
            if kind is KernelKind.CSR_INTRA_BLOCKED:
                _check_block_local(self.csr, self.block_size)
            launch_fused(self.csr, x, y, op, flags=flags, other_touched=other_touched, deg=deg,
                         gin_scale=g)
        elif kind is KernelKind.DENSE_BLOCK:
            if self.blocks is None:
                raise KernelError("dense_block kernel requires an intra subgraph")
            if op is AggregateOp.MAX:
                raise KernelError("dense_block kernel does not support max aggregation")
            if (op is AggregateOp.SUM and gin_scale is None
                    and dense_block_engine(self.blocks, x, None) == "tc"):
                # combine(sum): the inter partial already in y (0 where untouched)
                launch_dense_block_tc(self.blocks, x, y, beta=1.0)
            else:
                launch_dense_block(self.blocks, x, y, op, flags, other_touched, deg, g)
        else:
            mine = self.run(kind, x, op, tile_budget_bytes)
            other = PartialResult(values=y, touched=other_touched, op=op)
            y.copy_(combine(mine, other, op, full_in_degree=deg))
            if gin_scale is not None:
                y.copy_(np.float32(gin_scale) * x + y)


def decomposed_execs(d: DecomposedGraph) -> tuple[SubgraphExec, SubgraphExec]:
    """Formats of both roles, built once per DecomposedGraph and cached."""
    ex = d._cache.get("execs")
    if ex is None:
        ex = (SubgraphExec.for_intra(d.intra, d.block_size),
              SubgraphExec.for_inter(d.inter, d.block_size))
        d._cache["execs"] = ex
    return ex


CSR_KINDS = (KernelKind.CSR_INTRA_BLOCKED, KernelKind.CSR_INTER)


def fusable(kernel_intra: KernelKind, kernel_inter: KernelKind, block_size: int = 16) -> bool:
    """A CSR x CSR pair runs as ONE fused launch over the full CSR (same bits);
    so do (dense_block, csr_inter) for 16-row blocks (the slab kernel's
    dense-intra mode) and either intra kernel with coo_atomic as the inter
    role (AG_EPI_INTER_COO: the inter edges in any order, like the reference's
    scrambled fp64 bincount)."""
    if kernel_inter not in (KernelKind.CSR_INTER, KernelKind.COO_ATOMIC):
        return False
    return kernel_intra in CSR_KINDS or (kernel_intra is KernelKind.DENSE_BLOCK
                                         and block_size == 16)


def fused_ok(kernel_intra: KernelKind, kernel_inter: KernelKind, block_size: int,
             op: AggregateOp) -> bool:
    """fusable(), restricted to what the fused kernel computes for `op` (the
    dense-intra and order-free inter modes are sum-only; dense_block rejects
    max anyway)."""
    return fusable(kernel_intra, kernel_inter, block_size) and (
        op is AggregateOp.SUM or (kernel_intra is not KernelKind.DENSE_BLOCK
                                  and kernel_inter is not KernelKind.COO_ATOMIC))


def run_fused_pair(d: DecomposedGraph, x: torch.Tensor, y: torch.Tensor, op: AggregateOp,
                   gin_scale: float | None = None, relu_src: torch.Tensor | None = None,
                   relu: bool = False, dense_intra: bool = False,
                   kernel_intra: KernelKind | None = None,
                   kernel_inter: KernelKind = KernelKind.CSR_INTER,
                   relu_bits_in: torch.Tensor | None = None,
                   relu_out: torch.Tensor | None = None) -> None:
    """y = combine(intra, inter) [+ gin] [relu] [* (relu_src > 0)] in one pass
    over the full reordered CSR for the selector pair (kernel_intra,
    kernel_inter); `dense_intra` is shorthand for kernel_intra=dense_block.
    The ReLU-backward mask is relu_src (fp32) or relu_bits_in (bit mask);
    with relu=True, relu_out receives y's relu bits."""
    if kernel_intra is None:
        kernel_intra = KernelKind.DENSE_BLOCK if dense_intra else KernelKind.CSR_INTRA_BLOCKED
    if not fused_ok(kernel_intra, kernel_inter, d.block_size, op):
        raise KernelError(f"no fused kernel for ({kernel_intra.value}, {kernel_inter.value}, "
                          f"{op.value}, block_size={d.block_size})")
    full = full_graph(d)
    flags = ((_lib.AG_EPI_GIN if gin_scale is not None else 0)
             | (_lib.AG_EPI_RELU if relu else 0)
             | (_lib.AG_EPI_INTER_COO if kernel_inter is KernelKind.COO_ATOMIC else 0))
    launch_fused(to_csr(full), x, y, op, block=d.block_size, mask=3, flags=flags,
                 deg=d.full_in_degree, gin_scale=0.0 if gin_scale is None else gin_scale,
                 relu_src=relu_src, dense_intra=kernel_intra is KernelKind.DENSE_BLOCK,
                 relu_bits_in=relu_bits_in, relu_out=relu_out if relu else None)


def aggregate_full(g: Graph, x, op: AggregateOp, kernel: KernelKind = KernelKind.CSR_INTER,
                   threads: int = 1) -> torch.Tensor:
    """One kernel over the full graph, finalised as combine(partial, empty)."""
    del threads
    x = _check_features(g.num_vertices, x)
    if kernel is KernelKind.CSR_INTER:
        y = torch.empty((g.num_vertices, x.shape[1]), dtype=torch.float32, device=x.device)
        launch_fused(to_csr(g), x, y, op, flags=_lib.AG_EPI_COMBINE | _lib.AG_EPI_EMPTY_OTHER,
                     deg=g.in_degrees())
        return y
    ex = SubgraphExec.for_inter(g, block_size=max(g.num_vertices, 1))
    partial = ex.run(kernel, x, op)
    other = empty_partial(g.num_vertices, x.shape[1], op)
    return combine(partial, other, op, full_in_degree=g.in_degrees())


def aggregate_decomposed(d: DecomposedGraph, x, op: AggregateOp,
                         kernel_intra: KernelKind = KernelKind.CSR_INTRA_BLOCKED,
                         kernel_inter: KernelKind = KernelKind.COO_ATOMIC,
                         tile_budget_bytes: int = DEFAULT_TILE_BUDGET_BYTES,
                         threads: int = 1, gin_scale: float | None = None) -> torch.Tensor:
    """Aggregate a decomposed graph with one kernel per role (kernels.py:365-376).

    The inter kernel writes its raw partial, the intra kernel combines into
    it in its epilogue (and adds gin_scale * x when given, models.py:111).
    """
    del threads
    x = _check_features(d.num_vertices, x)
    y = torch.empty((d.num_vertices, x.shape[1]), dtype=torch.float32, device=x.device)
    if fused_ok(kernel_intra, kernel_inter, d.block_size, op):
        run_fused_pair(d, x, y, op, gin_scale, kernel_intra=kernel_intra,
                       kernel_inter=kernel_inter)
        return y
    intra, inter = decomposed_execs(d)
    inter.run_raw_into(kernel_inter, x, y, op, tile_budget_bytes)
    intra.run_combine_into(kernel_intra, x, y, op, inter.csr.touched(), d.full_in_degree,
                           tile_budget_bytes, gin_scale)
    return y
