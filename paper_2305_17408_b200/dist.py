"""Multi-GPU data path: 1-D community row partition, feature-halo all-gather,
weight-gradient all-reduce (north_star "Multi-GPU").

One process per GPU (torchrun), torch.distributed over NCCL for the plumbing.
The reordered graph's destination rows are cut into G contiguous ranges whose
boundaries are multiples of the community size B (so every diagonal block and
every intra edge is rank-local) and that are balanced by nnz + a per-row cost.
Rank k owns rows [b_k, b_{k+1}): their CSR rows (both roles, role-ordered
exactly as on one GPU), their feature rows, and the matching rows of the
transposed graph for the backward pass.

Halo.  need[(k, j)] is the sorted set of rank j's rows that rank k's edges
reference.  Every rank derives all of them from the (replicated) topology, so
the exchange is one uneven all-to-all per aggregation: rank j gathers
need[(k, j)] for every k into one send buffer, rank k receives them into the
tail of an *extended* feature matrix

    x_ext = [ x_local (n_k rows) | pad to a multiple of B | halo from rank 0 | rank 1 | ... ]

and the local CSR's columns are remapped into x_ext once, at build time
(local row r - b_k, or halo slot offset_j + position in need[(k, j)]).  Only
the rows a rank reads cross NVLink (the padded all-gather of the first
version delivered 5.9x that at G = 8; HaloPlan.stats reports both).  The
fused aggregation kernel then runs unchanged on the local rows: every
destination row is reduced entirely on its owner with the same per-row order,
so with the bitwise CSR pair the G-rank aggregation is BITWISE equal to the
1-GPU one.  dW is a sum of per-rank partial GEMMs, reduced with one bucketed
all-reduce (tolerance-level parity).

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
    (sorted global ids, int64, on col's device) -- what a padded all-gather
    would have to deliver to everyone."""
    need = peer_sets(row_ptr, col, bounds)
    G = len(bounds) - 1
    out = []
    for j in range(G):
        parts = [need[(k, j)] for k in range(G) if k != j]
        out.append(torch.unique(torch.cat(parts)) if parts else
                   torch.empty(0, dtype=torch.int64, device=col.device))
    return out


def peer_sets(row_ptr: torch.Tensor, col: torch.Tensor, bounds: list[int]) -> dict:
    """need[(k, j)] for every pair of ranks k != j: the sorted global ids of
    rank j's rows that rank k's rows reference -- exactly what j sends k."""
    dev = col.device
    V = row_ptr.numel() - 1
    G = len(bounds) - 1
    counts = (row_ptr[1:] - row_ptr[:-1]).to(torch.int64)
    dst_owner = torch.repeat_interleave(owner_of(torch.arange(V, device=dev), bounds), counts)
    src = col.to(torch.int64)
    src_owner = owner_of(src, bounds)
    remote = dst_owner != src_owner
    key = (dst_owner[remote] * G + src_owner[remote]) * (V + 1) + src[remote]
    key = torch.unique(key)  # sorted by (k, j), then source id
    pair, ids = key // (V + 1), key % (V + 1)
    sizes = torch.bincount(pair, minlength=G * G).tolist()
    chunks = torch.split(ids, sizes)
    return {(k, j): chunks[k * G + j] for k in range(G) for j in range(G) if k != j}


@dataclass
class HaloPlan:
    """One rank's view of the exchange for one topology (forward or transpose).

    x_ext = [ local rows (n_local) | pad to a multiple of B | halo ]: the halo
    holds, for every peer j in rank order, exactly the rows of j that this
    rank's edges reference (need[(rank, j)], sorted).  One uneven all-to-all
    per aggregation delivers them (no padding, no rows nobody asked for)."""

    rank: int
    world: int
    bounds: list
    block: int
    n_local: int
    halo_base: int             # first halo row in x_ext (multiple of B)
    recv_sets: list            # recv_sets[j]: global ids received from j (sorted)
    recv_counts: list          # |recv_sets[j]|
    send_counts: list          # rows this rank sends to each peer
    send_local: torch.Tensor   # int64[sum(send_counts)]: local rows to send, peer order
    allgather_rows: int        # rows a padded all-gather would deliver (G * max_j |S_j|)

    @property
    def ext_rows(self) -> int:
        return self.halo_base + sum(self.recv_counts)

    @property
    def recv_offsets(self) -> list:
        off, o = [], 0
        for c in self.recv_counts:
            off.append(o)
            o += c
        return off

    @classmethod
    def build(cls, row_ptr, col, bounds, rank: int, block: int) -> "HaloPlan":
        world = len(bounds) - 1
        need = peer_sets(row_ptr, col, bounds)
        dev = col.device
        empty = torch.empty(0, dtype=torch.int64, device=dev)
        r0, r1 = bounds[rank], bounds[rank + 1]
        recv_sets = [need.get((rank, j), empty) for j in range(world)]
        sends = [need.get((j, rank), empty) - r0 for j in range(world)]
        smax = 0
        for j in range(world):
            parts = [need[(k, j)] for k in range(world) if k != j]
            if parts:
                smax = max(smax, int(torch.unique(torch.cat(parts)).numel()))
        n_local = r1 - r0
        return cls(rank=rank, world=world, bounds=list(bounds), block=block, n_local=n_local,
                   halo_base=math.ceil(n_local / block) * block, recv_sets=recv_sets,
                   recv_counts=[int(t.numel()) for t in recv_sets],
                   send_counts=[int(t.numel()) for t in sends],
                   send_local=torch.cat(sends) if sends else empty,
                   allgather_rows=world * smax if world > 1 else 0)

    def remap(self, cols: torch.Tensor) -> torch.Tensor:
        """Global source ids -> rows of x_ext (int32)."""
        c = cols.to(torch.int64)
        r0, r1 = self.bounds[self.rank], self.bounds[self.rank + 1]
        out = torch.empty_like(c)
        local = (c >= r0) & (c < r1)
        out[local] = c[local] - r0
        own = owner_of(c, self.bounds)
        offs = self.recv_offsets
        for j in range(self.world):
            m = (~local) & (own == j)
            if not bool(m.any()):
                continue
            S = self.recv_sets[j]
            pos = torch.searchsorted(S, c[m])
            if S.numel() == 0 or not bool(torch.equal(S[pos.clamp(max=S.numel() - 1)], c[m])):
                raise RuntimeError("halo plan does not cover a referenced row")
            out[m] = self.halo_base + offs[j] + pos
        return out.to(torch.int32)

    def new_ext(self, feat: int, device, dtype=torch.float32) -> torch.Tensor:
        return torch.empty((self.ext_rows, feat), dtype=dtype, device=device)

    def stats(self) -> dict:
        """Halo rows this rank needs (= receives) vs what the padded all-gather
        of the previous design delivered."""
        return {"rank": self.rank, "n_local": self.n_local, "halo_rows": sum(self.recv_counts),
                "sent_rows": sum(self.send_counts), "allgather_rows": self.allgather_rows}

    def exchange(self, x_ext: torch.Tensor, group=None, async_op: bool = False):
        """Fill x_ext's halo rows from the peers (x_ext[:n_local] must hold
        this rank's rows): one uneven all-to-all.  async_op: returns the work
        handle (wait() before reading the halo) so independent work overlaps."""
        if self.world == 1 or (sum(self.recv_counts) == 0 and sum(self.send_counts) == 0):
            return None
        send = x_ext.index_select(0, self.send_local)
        recv = x_ext[self.halo_base:self.ext_rows]
        return dist.all_to_all_single(recv, send, output_split_sizes=self.recv_counts,
                                      input_split_sizes=self.send_counts, group=group,
                                      async_op=async_op)


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
PAIRS = ("dense_coo", "csr")  # fused selector pairs DistGNN can run per aggregation


class TorchComm:
    """DistGNN's collectives over torch.distributed (NCCL on the GPU box).
    Tests substitute an in-process implementation with the same methods."""

    def __init__(self, group=None):
        self.group = group

    def exchange(self, plan: HaloPlan, x_ext: torch.Tensor, async_op: bool = False):
        return plan.exchange(x_ext, self.group, async_op=async_op)

    def all_reduce(self, t: torch.Tensor, op=None) -> None:
        if op is None:
            dist.all_reduce(t, group=self.group)
        else:
            dist.all_reduce(t, op=op, group=self.group)


class DistGNN:
    """Row-partitioned GCN / GIN training step on one rank (GPU path).

    The same composition as models.GNN over this rank's rows,
    including its reassociation: a narrowing layer runs its update GEMM on the
    local rows first and exchanges / aggregates the narrow product (so the
    halo carries the narrow width too).  Aggregations run the fused kernel on
    the halo-extended features with a selector pair per (direction, width):
    "dense_coo" (dense_block intra + coo_atomic inter, the pair the 1-GPU
    autotune picks at every C5 width) or "csr" (both CSR roles, bitwise);
    autotune() times both on the rank's operators, all ranks agreeing on the
    slowest rank's timing.  In the backward pass the halo exchange of d(A H)
    runs asynchronously under the layer's dW GEMM.  dW partials are bucketed
    into one flat buffer and all-reduced; the loss is a sum of per-rank
    partials over the GLOBAL masked count.  Weights are replicated (identical
    seeds on every rank)."""

    def __init__(self, model: str, dims, fwd: LocalOperator, bwd: LocalOperator, weights,
                 gin_eps: float = 0.0, group=None, pair: str = "dense_coo",
                 reassociate: bool = True):
        from . import models
        if pair not in PAIRS:
            raise ValueError(f"pair must be one of {PAIRS}")
        self.model, self.dims = model, list(dims)
        self.fwd, self.bwd = fwd, bwd
        self.weights = weights
        self.gin_eps = gin_eps
        self.group = group
        self.default_pair = pair
        self.kernels = {}  # (direction, width) -> pair name (autotune)
        self.reassociate = reassociate
        dev = weights[0].device
        sizes = [w.shape[0] * models._pad4(w.shape[1]) for w in weights]
        self.flat = torch.zeros(sum(sizes), dtype=torch.float32, device=dev)
        self.grads, off = [], 0
        for w, n in zip(weights, sizes):
            buf = self.flat[off:off + n].view(w.shape[0], models._pad4(w.shape[1]))
            self.grads.append(buf[:, :w.shape[1]])
            off += n
        self.events = None
        self._dense = {}
        self.comm = TorchComm(group)

    @classmethod
    def build(cls, model: str, dims, subject, rank: int, world: int, seed: int = 0,
              gin_eps: float = 0.0, group=None, subject_t=None, pair: str = "dense_coo",
              reassociate: bool = True) -> "DistGNN":
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
        net = cls(model, dims, ops[0], ops[1], local.weights, gin_eps, group, pair=pair,
                  reassociate=reassociate)
        net.bounds = bounds
        return net

    @property
    def num_layers(self) -> int:
        return len(self.dims) - 1

    def gemm_first(self, l: int) -> bool:
        return self.reassociate and self.dims[l + 1] < self.dims[l]

    def gin_scale(self):
        import numpy as np
        return float(np.float32(1.0 + self.gin_eps)) if self.model == "gin" else None

    def dense_blocks(self, op: LocalOperator) -> torch.Tensor:
        """The local operator's intra runs as dense 16 x 16 blocks (B = 16;
        rank ranges are 16-aligned, so local block k is global block k + b/16)."""
        w = self._dense.get(id(op))
        if w is None:
            from . import _lib
            nb = max((op.num_rows + 15) // 16, 1)
            w = torch.empty(nb * 256, dtype=torch.float32, device=op.col.device)
            _lib.call("ag_slab_dense_blocks", op.num_rows, _lib.ptr(op.row_ptr), _lib.ptr(op.mid),
                      _lib.ptr(op.col), _lib.ptr(op.val), _lib.ptr(w), _lib.stream())
            self._dense[id(op)] = w
        return w

    def pair(self, direction: str, feat: int) -> str:
        return self.kernels.get((direction, feat), self.default_pair)

    def aggregate(self, op: LocalOperator, x_ext: torch.Tensor, direction: str = "fwd",
                  relu_bits=None, relu: bool = False, relu_out=None, relu_src=None,
                  pair: str | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
        """This rank's rows of A_hat x (x_ext: halo exchanged; row stride =
        width).  relu_bits / relu_src: the ReLU backward of the layer below
        (bit mask / fp32); relu: the forward activation, its bits to relu_out."""
        from . import _lib
        from .kernels import relu_bits as make_bits
        F = x_ext.shape[1]
        pair = pair or self.pair(direction, F)
        dense = pair == "dense_coo" and op.mid is not None and self.fwd.plan.block == 16
        if out is None:
            out = torch.empty((op.num_rows, F), dtype=torch.float32, device=x_ext.device)
        elif tuple(out.shape) != (op.num_rows, F) or out.stride(0) != F:
            raise ValueError("out must be a contiguous [rows, width] block")
        gs = self.gin_scale()
        if relu_bits is None and relu_src is not None:
            relu_bits = make_bits(relu_src)
        flags = ((_lib.AG_EPI_GIN if gs is not None else 0)
                 | (_lib.AG_EPI_RELU_MASK if relu_bits is not None else 0)
                 | (_lib.AG_EPI_RELU if relu else 0)
                 | (_lib.AG_EPI_INTER_COO if dense else 0))
        e0 = e1 = None
        if self.events is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
        _lib.call("ag_fused_spmm", op.num_rows, F, 3 if op.mid is not None else 2,
                  _lib.ptr(op.row_ptr), _lib.ptr(op.mid), *map(_lib.ptr, op.codes()),
                  int(op.val is not None), _lib.ptr(self.dense_blocks(op)) if dense else None,
                  op.num_edges, _lib.ptr(x_ext), _lib.ptr(out), _lib.AG_OP["sum"], flags, None,
                  _lib.ptr(op.deg), 0.0 if gs is None else gs, _lib.ptr(relu_bits),
                  _lib.ptr(relu_out if relu else None), x_ext.shape[0], op.window(),
                  _lib.stream())
        if e0 is not None:
            e1.record()
            self.events.append((e0, e1, F, op))
        return out

    def autotune(self, reps: int = 5) -> dict:
        """Pick the fused pair per (direction, width) this step aggregates at:
        each candidate timed on this rank's operator, the per-candidate MAX
        over ranks compared (every rank picks the same pair)."""
        from . import models
        from .models import _time_ms
        widths = {"fwd": set(), "bwd": set()}
        for l in range(self.num_layers):
            if self.gemm_first(l):
                widths["fwd"].add(models._pad4(self.dims[l + 1]))
                widths["bwd"].add(models._pad4(self.dims[l + 1]))
            else:
                widths["fwd"].add(models._pad4(self.dims[l]))
                if l > 0:
                    widths["bwd"].add(models._pad4(self.dims[l]))
        for direction, op in (("fwd", self.fwd), ("bwd", self.bwd)):
            for f in sorted(widths[direction]):
                x_ext = torch.randn((op.plan.ext_rows, f), device=op.col.device)
                ts = torch.tensor([_time_ms(lambda: self.aggregate(op, x_ext, direction, pair=p),
                                            reps=reps) for p in PAIRS],
                                  dtype=torch.float64, device=op.col.device)
                if op.plan.world > 1:
                    self.comm.all_reduce(ts, op=dist.ReduceOp.MAX)
                self.kernels[(direction, f)] = PAIRS[int(torch.argmin(ts).item())]
        return dict(self.kernels)

    def input_ext(self, x_local: torch.Tensor) -> torch.Tensor:
        """Extended layer-0 features from this rank's rows (copy; the halo is
        exchanged by train_step)."""
        from . import models
        F = x_local.shape[1]
        ext = self.fwd.plan.new_ext(models._pad4(F), x_local.device)
        ext[:self.fwd.num_rows, :F].copy_(x_local, non_blocking=True)
        if models._pad4(F) != F:
            ext[:, F:].zero_()
        return ext

    def _ext(self, plan: HaloPlan, width: int, dev) -> torch.Tensor:
        """[ext_rows, pad4(width)] buffer (the halo rows filled by exchange)."""
        from . import models
        return plan.new_ext(models._pad4(width), dev)

    def train_step(self, x_ext, labels, mask, num_masked: int, lr: float = 0.01):
        """One epoch on this rank's rows.  x_ext: input_ext(...) (halo not yet
        exchanged); labels/mask: local rows; num_masked: GLOBAL count."""
        from . import _lib, models
        from .kernels import gemm, relu_bits_empty
        n = self.fwd.num_rows
        L = self.num_layers
        dev = x_ext.device
        saved = []
        h_ext, width = x_ext, self.dims[0]
        for l in range(L):
            last = l == L - 1
            dout = self.dims[l + 1]
            bits = None if last else relu_bits_empty(n, models._pad4(dout), dev)
            if self.gemm_first(l):
                # P = H W on the local rows, exchange the narrow P, A_hat P (+ GIN)
                p_ext = self._ext(self.fwd.plan, dout, dev)
                if models._pad4(dout) != dout:
                    p_ext[:n, dout:].zero_()
                gemm(h_ext[:n, :width], self.weights[l], p_ext[:n, :dout])
                self.comm.exchange(self.fwd.plan, p_ext)
                # an aggregate-first layer above exchanges this output: write it
                # straight into the rows of an extended buffer
                h_next = None if last or self.gemm_first(l + 1) else \
                    self._ext(self.fwd.plan, dout, dev)
                out = self.aggregate(self.fwd, p_ext, "fwd", relu=not last, relu_out=bits,
                                     out=None if h_next is None else h_next[:n])
                saved.append(("gemm", h_ext[:n, :width], out[:, :dout], bits))
                if h_next is None:
                    h_next = out
            else:
                self.comm.exchange(self.fwd.plan, h_ext)
                agg = self.aggregate(self.fwd, h_ext, "fwd")
                out_ext = self._ext(self.fwd.plan, dout, dev)
                gemm(agg[:, :width], self.weights[l], out_ext[:n, :dout], relu=not last,
                     mask_out=bits)
                saved.append(("agg", agg[:, :width], out_ext[:n, :dout], bits))
                h_next = out_ext
            h_ext, width = h_next, dout
        logits = h_ext[:n, :width]
        loss = torch.empty(1, dtype=torch.float32, device=dev)
        g = torch.empty((n, models._pad4(width)), dtype=torch.float32, device=dev)[:, :width]  # xent writes the pad
        _lib.call("ag_softmax_xent", n, logits.shape[1], logits.stride(0), _lib.ptr(logits),
                  _lib.ptr(labels), _lib.ptr(mask), int(num_masked), _lib.ptr(loss),
                  _lib.ptr(g), g.stride(0), _lib.stream())
        for l in range(L - 1, -1, -1):
            kind, operand, _, _ = saved[l]
            bits_prev = saved[l - 1][3] if l > 0 else None
            din, dout = self.dims[l], self.dims[l + 1]
            if kind == "agg":
                work = d_ext = None
                if l > 0:  # d(A H) = g W^T, exchanged under the dW GEMM
                    d_ext = self._ext(self.bwd.plan, din, dev)
                    if models._pad4(din) != din:
                        d_ext[:n, din:].zero_()
                    gemm(g, self.weights[l], d_ext[:n, :din], trans_b=True)
                    work = self.comm.exchange(self.bwd.plan, d_ext, async_op=True)
                gemm(operand, g, self.grads[l], trans_a=True)                   # dW = (A H)^T g
                if l == 0:
                    break
                if work is not None:
                    work.wait()
                g = self.aggregate(self.bwd, d_ext, "bwd", relu_bits=bits_prev)[:, :din]
            else:
                g_ext = self._ext(self.bwd.plan, dout, dev)
                g_ext[:n].zero_()
                g_ext[:n, :dout].copy_(g)
                self.comm.exchange(self.bwd.plan, g_ext)
                q = self.aggregate(self.bwd, g_ext, "bwd")[:, :dout]
                gemm(operand, q, self.grads[l], trans_a=True)                   # dW = H^T q
                if l == 0:
                    break
                g = models._padded_empty(n, din, dev)
                gemm(q, self.weights[l], g, trans_b=True, relu_mask_bits=bits_prev)  # dH, ReLU bwd
        if self.bwd.plan.world > 1:
            self.comm.all_reduce(self.flat)  # every dW in one bucket
            self.comm.all_reduce(loss)
        for w, dw in zip(self.weights, self.grads):
            wb, gb = models._base(w), models._base(dw)
            _lib.call("ag_sgd_step", wb.numel(), _lib.ptr(wb), _lib.ptr(gb), float(lr),
                      _lib.stream())
        return loss, self.grads
