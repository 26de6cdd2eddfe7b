"""Multi-GPU data path: 1-D community row partition, feature-halo all-gather,
weight-gradient all-reduce (north_star "Multi-GPU").

One process per GPU (torchrun), torch.distributed over NCCL for the plumbing.
The reordered graph's destination rows are cut into G contiguous ranges whose
boundaries are multiples of the community size B (so every diagonal block and
every intra edge is rank-local) and that are balanced by nnz + a per-row cost.
Rank k owns rows [b_k, b_{k+1}): their CSR rows (both roles, role-ordered
exactly as on one GPU), their feature rows, and the matching rows of the
transposed graph for the backward pass.

Halo.  Rank j's *send set* S_j is the sorted set of its rows that some edge of
another rank references.  Every rank derives all S_j from the (replicated)
topology, so the exchange is one fixed-size collective per aggregation:
``all_gather`` of the [max_j |S_j|, F] send buffers into the tail of an
*extended* feature matrix

    x_ext = [ x_local (n_k rows) | pad to a multiple of B | halo (G * max|S| rows) ]

and the local CSR's columns are remapped into x_ext once, at build time
(local row r - b_k, or halo slot j * max|S| + position in S_j).  The fused
aggregation kernel then runs unchanged on the local rows: every destination
row is reduced entirely on its owner with the same per-row order, so the
G-rank aggregation is BITWISE equal to the 1-GPU one.  dW is a sum of per-rank
partial GEMMs, reduced with one bucketed all-reduce (tolerance-level parity).

The host logic (partition, send sets, remap, exchange) is plain torch and runs
on CPU tensors too, so the world-size-2 gloo tests exercise it without a GPU.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.distributed as dist

ROW_COST = 4  # a row's fixed cost in edge units (epilogue + topology), as in the kernel


def balanced_bounds(row_ptr: torch.Tensor, world: int, block: int) -> list[int]:
    """B-aligned row boundaries [0 = b_0 <= ... <= b_G = V] balancing
    nnz + ROW_COST * rows (deterministic: every rank computes the same cut)."""
    rp = row_ptr.to("cpu", torch.int64)
    V = rp.numel() - 1
    if world < 1:
        raise ValueError("world size must be >= 1")
    cost = rp + ROW_COST * torch.arange(V + 1, dtype=torch.int64)
    total = int(cost[-1])
    bounds = [0]
    for k in range(1, world):
        target = total * k // world
        r = int(torch.searchsorted(cost, torch.tensor([target])).item())
        r = min(V, int(round(r / block)) * block)
        bounds.append(max(bounds[-1], r))
    bounds.append(V)
    return bounds


def owner_of(ids: torch.Tensor, bounds: list[int]) -> torch.Tensor:
    b = torch.tensor(bounds[1:-1], dtype=torch.int64, device=ids.device)
    return torch.bucketize(ids.to(torch.int64), b, right=True)


def send_sets(row_ptr: torch.Tensor, col: torch.Tensor, bounds: list[int]) -> list[torch.Tensor]:
    """S_j for every rank j: rows of j's range referenced by other ranks' rows
    (sorted global ids, int64, on col's device)."""
    dev = col.device
    V = row_ptr.numel() - 1
    counts = (row_ptr[1:] - row_ptr[:-1]).to(torch.int64)
    dst_owner = torch.repeat_interleave(owner_of(torch.arange(V, device=dev), bounds), counts)
    src = col.to(torch.int64)
    src_owner = owner_of(src, bounds)
    remote = dst_owner != src_owner
    out = []
    for j in range(len(bounds) - 1):
        sel = src[remote & (src_owner == j)]
        out.append(torch.unique(sel))  # sorted
    return out


@dataclass
class HaloPlan:
    """One rank's view of the exchange for one topology (forward or transpose)."""

    rank: int
    world: int
    bounds: list
    block: int
    n_local: int
    halo_base: int            # first halo row in x_ext (multiple of B)
    max_send: int             # rows per rank in the all-gather (padded)
    send_local: torch.Tensor  # int64[max_send]: local rows this rank sends (padded with 0)
    sets: list                # S_j (global ids) for every j

    @property
    def ext_rows(self) -> int:
        return self.halo_base + self.world * self.max_send

    @classmethod
    def build(cls, row_ptr, col, bounds, rank: int, block: int) -> "HaloPlan":
        world = len(bounds) - 1
        sets = send_sets(row_ptr, col, bounds)
        max_send = max([int(s.numel()) for s in sets] + [0])
        r0, r1 = bounds[rank], bounds[rank + 1]
        n_local = r1 - r0
        halo_base = math.ceil(n_local / block) * block
        send = torch.zeros(max_send, dtype=torch.int64, device=col.device)
        mine = sets[rank]
        send[:mine.numel()] = mine - r0
        return cls(rank=rank, world=world, bounds=list(bounds), block=block, n_local=n_local,
                   halo_base=halo_base, max_send=max_send, send_local=send, sets=sets)

    def remap(self, cols: torch.Tensor) -> torch.Tensor:
        """Global source ids -> rows of x_ext (int32)."""
        c = cols.to(torch.int64)
        r0, r1 = self.bounds[self.rank], self.bounds[self.rank + 1]
        out = torch.empty_like(c)
        local = (c >= r0) & (c < r1)
        out[local] = c[local] - r0
        own = owner_of(c, self.bounds)
        for j in range(self.world):
            m = (~local) & (own == j)
            if not bool(m.any()):
                continue
            pos = torch.searchsorted(self.sets[j], c[m])
            if not bool(torch.equal(self.sets[j][pos.clamp(max=self.sets[j].numel() - 1)], c[m])):
                raise RuntimeError("halo plan does not cover a referenced row")
            out[m] = self.halo_base + j * self.max_send + pos
        return out.to(torch.int32)

    def new_ext(self, feat: int, device, dtype=torch.float32) -> torch.Tensor:
        return torch.empty((self.ext_rows, feat), dtype=dtype, device=device)

    def exchange(self, x_ext: torch.Tensor, group=None) -> None:
        """Fill x_ext's halo rows from the other ranks (x_ext[:n_local] must
        hold this rank's rows).  One all-gather of max_send rows per rank."""
        if self.world == 1 or self.max_send == 0:
            return
        send = x_ext.index_select(0, self.send_local)
        recv = x_ext[self.halo_base:self.halo_base + self.world * self.max_send]
        all_gather_rows(recv, send, group)


def all_gather_rows(recv: torch.Tensor, send: torch.Tensor, group=None) -> None:
    """recv[j*n:(j+1)*n] = send of rank j (NCCL: one all_gather_into_tensor)."""
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(recv, send.contiguous(), group=group)
    else:  # gloo (CPU tests): list form
        n = send.shape[0]
        chunks = [torch.empty_like(send) for _ in range(dist.get_world_size(group))]
        dist.all_gather(chunks, send.contiguous(), group=group)
        for j, c in enumerate(chunks):
            recv[j * n:(j + 1) * n].copy_(c)


@dataclass
class LocalOperator:
    """This rank's rows of one (role-ordered) aggregation operator, columns
    remapped into the extended feature matrix of its HaloPlan."""

    plan: HaloPlan
    row_ptr: torch.Tensor          # int32[n_local + 1]
    mid: torch.Tensor | None       # int32[n_local] end of each row's intra run
    col: torch.Tensor              # int32[E_local] rows of x_ext
    val: torch.Tensor | None       # f32[E_local]
    deg: torch.Tensor | None       # int64[n_local] full in-degree (mean)

    @property
    def num_rows(self) -> int:
        return self.plan.n_local

    def window(self) -> int:
        """Slab-kernel ring radius over the local operator (halo rows sit
        past the local ones, so they read as far sources)."""
        w = getattr(self, "_window", None)
        if w is None:
            from . import _lib
            from .formats import SLAB_COVERAGE
            o = _lib.out_i32()
            _lib.call("ag_slab_window", self.num_rows, _lib.ptr(self.row_ptr), _lib.ptr(self.col),
                      SLAB_COVERAGE, _lib.byref(o), _lib.stream())
            w = int(o.value)
            object.__setattr__(self, "_window", w)
        return w

    def codes(self):
        """The slab layout of this operator for window(): (cv, rowinfo, far_cnt, far_src)."""
        c = getattr(self, "_codes", None)
        if c is None:
            from .formats import slab_codes
            c = slab_codes(self.num_rows, self.row_ptr, self.col, self.val, self.mid,
                           self.window())
            object.__setattr__(self, "_codes", c)
        return c

    @property
    def num_edges(self) -> int:
        return int(self.col.numel())

    @classmethod
    def build(cls, row_ptr, col, val, bounds, rank: int, block: int, mid=None, role_col=None,
              role_val=None, deg=None) -> "LocalOperator":
        """row_ptr/col are the plain CSR (for the send sets); mid/role_col/
        role_val the role-ordered copy (if None the plain CSR is one role)."""
        plan = HaloPlan.build(row_ptr, col, bounds, rank, block)
        r0, r1 = bounds[rank], bounds[rank + 1]
        e0, e1 = int(row_ptr[r0]), int(row_ptr[r1])
        rp = (row_ptr[r0:r1 + 1].to(torch.int64) - e0).to(torch.int32)
        cols = role_col if role_col is not None else col
        vals = role_val if role_col is not None else val
        lm = None if mid is None else (mid[r0:r1].to(torch.int64) - e0).to(torch.int32)
        lv = None if vals is None else vals[e0:e1].contiguous()
        ld = None if deg is None else deg[r0:r1].contiguous()
        return cls(plan=plan, row_ptr=rp.contiguous(), mid=lm, col=plan.remap(cols[e0:e1]),
                   val=lv, deg=ld)


# ------------------------------------------------------------ GPU training --
class DistGNN:
    """Row-partitioned GCN / GIN training step on one rank (GPU path).

    Same composition as models.GNN over this rank's rows:
    forward aggregations read the halo-extended activations, the update GEMMs
    run on local rows, dW partials are bucketed into one flat buffer and
    all-reduced, the loss is a sum of per-rank partials over the GLOBAL masked
    count.  Weights are replicated (identical seeds on every rank)."""

    def __init__(self, model: str, dims, fwd: LocalOperator, bwd: LocalOperator, weights,
                 gin_eps: float = 0.0, group=None):
        from . import models
        self.model, self.dims = model, list(dims)
        self.fwd, self.bwd = fwd, bwd
        self.weights = weights
        self.gin_eps = gin_eps
        self.group = group
        dev = weights[0].device
        sizes = [w.shape[0] * models._pad4(w.shape[1]) for w in weights]
        self.flat = torch.zeros(sum(sizes), dtype=torch.float32, device=dev)
        self.grads, off = [], 0
        for w, n in zip(weights, sizes):
            buf = self.flat[off:off + n].view(w.shape[0], models._pad4(w.shape[1]))
            self.grads.append(buf[:, :w.shape[1]])
            off += n
        self.events = None

    @classmethod
    def build(cls, model: str, dims, subject, rank: int, world: int, seed: int = 0,
              gin_eps: float = 0.0, group=None, subject_t=None) -> "DistGNN":
        """subject: the DecomposedGraph of the full reordered graph (every rank
        holds the topology; only its rows' operators stay on the device)."""
        from . import models
        from .decompose import decompose, full_graph
        from .formats import to_csr
        if subject_t is None:
            subject_t = decompose(full_graph(subject).reverse(), subject.block_size)
        B = subject.block_size
        ops = []
        for sub in (subject, subject_t):
            csr = to_csr(full_graph(sub))
            mid, rcol, rval = csr.role_layout(B)
            if not ops:
                bounds = balanced_bounds(csr.row_ptr, world, B)
            ops.append(LocalOperator.build(csr.row_ptr, csr.col_idx, csr.kernel_val, bounds,
                                           rank, B, mid=mid, role_col=rcol, role_val=rval,
                                           deg=sub.full_in_degree))
        local = models.GNN.build(model, dims, subject, seed=seed, gin_eps=gin_eps,
                                 subject_t=subject_t)
        net = cls(model, dims, ops[0], ops[1], local.weights, gin_eps, group)
        net.bounds = bounds
        return net

    def gin_scale(self):
        import numpy as np
        return float(np.float32(1.0 + self.gin_eps)) if self.model == "gin" else None

    def aggregate(self, op: LocalOperator, x_ext: torch.Tensor, relu_src=None) -> torch.Tensor:
        from . import _lib
        F = x_ext.shape[1]
        out = torch.empty((op.num_rows, F), dtype=torch.float32, device=x_ext.device)
        gs = self.gin_scale()
        flags = (_lib.AG_EPI_GIN if gs is not None else 0) | \
            (_lib.AG_EPI_RELU_MASK if relu_src is not None else 0)
        rbits = None
        if relu_src is not None:  # the kernel reads the layer's bit-packed ReLU mask
            from .kernels import relu_bits
            rbits = relu_bits(relu_src)
        e0 = e1 = None
        if self.events is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
        _lib.call("ag_fused_spmm", op.num_rows, F, 3 if op.mid is not None else 2,
                  _lib.ptr(op.row_ptr), _lib.ptr(op.mid), *map(_lib.ptr, op.codes()),
                  int(op.val is not None), None,
                  op.num_edges, _lib.ptr(x_ext), _lib.ptr(out), _lib.AG_OP["sum"], flags, None,
                  _lib.ptr(op.deg), 0.0 if gs is None else gs, _lib.ptr(rbits), None,
                  x_ext.shape[0], op.window(), _lib.stream())
        if e0 is not None:
            e1.record()
            self.events.append((e0, e1, F, op))
        return out

    def input_ext(self, x_local: torch.Tensor) -> torch.Tensor:
        """Extended layer-0 features from this rank's rows (copy + exchange)."""
        ext = self.fwd.plan.new_ext(x_local.shape[1], x_local.device)
        ext[:self.fwd.num_rows].copy_(x_local, non_blocking=True)
        return ext

    def train_step(self, x_ext, labels, mask, num_masked: int, lr: float = 0.01):
        """One epoch on this rank's rows.  x_ext: input_ext(...) (halo not yet
        exchanged); labels/mask: local rows; num_masked: GLOBAL count."""
        from . import _lib, models
        from .kernels import gemm
        n = self.fwd.num_rows
        L = len(self.dims) - 1
        saved = []
        h_ext = x_ext
        for l in range(L):
            self.fwd.plan.exchange(h_ext, self.group)
            agg = self.aggregate(self.fwd, h_ext)
            last = l == L - 1
            if last:
                out = models._padded_empty(n, self.dims[l + 1], agg.device)
                gemm(agg, self.weights[l], out)
            else:
                out = self.fwd.plan.new_ext(self.dims[l + 1], agg.device)
                gemm(agg, self.weights[l], out[:n], relu=True)
            saved.append((agg, out))
            h_ext = out
        logits = h_ext
        loss = torch.empty(1, dtype=torch.float32, device=logits.device)
        g = models._padded_empty(n, logits.shape[1], logits.device)
        _lib.call("ag_softmax_xent", n, logits.shape[1], logits.stride(0), _lib.ptr(logits),
                  _lib.ptr(labels), _lib.ptr(mask), int(num_masked), _lib.ptr(loss),
                  _lib.ptr(g), g.stride(0), _lib.stream())
        for l in range(L - 1, -1, -1):
            agg, _ = saved[l]
            gemm(agg, g, self.grads[l], trans_a=True)
            if l == 0:
                break
            d_ext = self.bwd.plan.new_ext(self.dims[l], agg.device)
            gemm(g, self.weights[l], d_ext[:n], trans_b=True)
            self.bwd.plan.exchange(d_ext, self.group)
            _, h_prev = saved[l - 1]
            g = self.aggregate(self.bwd, d_ext, relu_src=h_prev[:n])
        if self.bwd.plan.world > 1:
            dist.all_reduce(self.flat, group=self.group)  # every dW in one bucket
            dist.all_reduce(loss, group=self.group)
        for w, dw in zip(self.weights, self.grads):
            wb, gb = models._base(w), models._base(dw)
            _lib.call("ag_sgd_step", wb.numel(), _lib.ptr(wb), _lib.ptr(gb), float(lr),
                      _lib.stream())
        return loss, self.grads
