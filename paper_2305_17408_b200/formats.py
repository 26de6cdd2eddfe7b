"""Device-resident physical formats (reference formats.py:16-161).

CSR over destinations (row_ptr int32[V+1], col_idx int32[E], val f32[E]),
canonical COO (row, col, val) and per-community dense diagonal blocks.  All
are built on the device once per graph and cached (the reference rebuilds
them on every aggregate_decomposed call).  For unweighted
graphs the value array is implicit (the kernels take val=NULL, i.e. 1.0),
so GIN aggregation never reads a ones vector from HBM; `.val` materialises
it lazily for API compatibility.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .graph import Graph, as_device

# fraction of the (largest-ring-coverable) edges the slab kernel's ring must hold
SLAB_COVERAGE = 0.995


class CooMatrix:
    """Coordinate-format adjacency sorted by (row, col)."""

    __slots__ = ("num_vertices", "row", "col", "_val", "_ones", "_row_ptr")

    def __init__(self, num_vertices: int, row: torch.Tensor, col: torch.Tensor,
                 val: torch.Tensor | None):
        self.num_vertices = int(num_vertices)
        self.row, self.col, self._val, self._ones = row, col, val, None
        self._row_ptr = None

    @property
    def row_ptr(self) -> torch.Tensor:
        """Offsets of each destination's run (the rows are sorted), built once."""
        if self._row_ptr is None:
            rp = torch.empty(self.num_vertices + 1, dtype=torch.int32, device=self.row.device)
            _lib.call("ag_build_row_ptr", self.num_vertices, self.num_edges, _lib.ptr(self.row),
                      _lib.ptr(rp), _lib.stream())
            self._row_ptr = rp
        return self._row_ptr

    @property
    def val(self) -> torch.Tensor:
        if self._val is not None:
            return self._val
        if self._ones is None:
            self._ones = torch.ones(self.num_edges, dtype=torch.float32, device=self.row.device)
        return self._ones

    @property
    def kernel_val(self) -> torch.Tensor | None:
        return self._val

    @property
    def num_edges(self) -> int:
        return int(self.row.numel())


def slab_codes(num_rows: int, row_ptr: torch.Tensor, col: torch.Tensor, val, mid, window: int):
    """ag_slab_codes: (cv int32[2E], rowinfo int32[4V], far_cnt int32[nb],
    far_src int32[nb * cap])."""
    dev = row_ptr.device
    V = int(num_rows)
    nb = (V + 15) // 16
    cap = int(_lib.load().ag_slab_far_capacity())
    cv = torch.empty(max(2 * col.numel(), 2), dtype=torch.int32, device=dev)
    rowinfo = torch.empty(max(4 * V, 4), dtype=torch.int32, device=dev)
    far_cnt = torch.empty(max(nb, 1), dtype=torch.int32, device=dev)
    far_src = torch.empty(max(nb * cap, 1), dtype=torch.int32, device=dev)
    _lib.call("ag_slab_codes", V, _lib.ptr(row_ptr), _lib.ptr(col), _lib.ptr(val), _lib.ptr(mid),
              int(window), _lib.ptr(cv), _lib.ptr(rowinfo), _lib.ptr(far_cnt), _lib.ptr(far_src),
              _lib.stream())
    return cv, rowinfo, far_cnt, far_src


class CsrMatrix:
    """Compressed sparse rows over destination vertices."""

    __slots__ = ("num_vertices", "row_ptr", "col_idx", "_val", "_ones", "_rows", "_touched",
                 "_off_block", "_long", "_window", "_codes", "_dense16", "_band", "_ring_cov")

    def __init__(self, num_vertices: int, row_ptr: torch.Tensor, col_idx: torch.Tensor,
                 val: torch.Tensor | None, rows: torch.Tensor | None = None):
        self.num_vertices = int(num_vertices)
        self.row_ptr, self.col_idx, self._val, self._ones = row_ptr, col_idx, val, None
        self._rows = rows
        self._touched = None
        self._off_block: dict[int, int] = {}
        self._long = None
        self._window = None
        self._codes = {}
        self._dense16 = None
        self._band = None
        self._ring_cov = None

    @property
    def val(self) -> torch.Tensor:
        if self._val is not None:
            return self._val
        if self._ones is None:
            self._ones = torch.ones(self.num_edges, dtype=torch.float32,
                                    device=self.col_idx.device)
        return self._ones

    @property
    def kernel_val(self) -> torch.Tensor | None:
        return self._val

    @property
    def num_edges(self) -> int:
        return int(self.col_idx.numel())

    def window(self) -> int:
        """Ring radius (16-row blocks) of the slab aggregation kernel over this
        topology, picked once from the edge-distance histogram (ag_slab_window)."""
        if self._window is None:
            w = _lib.out_i32()
            _lib.call("ag_slab_window", self.num_vertices, _lib.ptr(self.row_ptr),
                      _lib.ptr(self.col_idx), SLAB_COVERAGE, _lib.byref(w), _lib.stream())
            self._window = int(w.value)
        return self._window

    def ring_coverage(self) -> float:
        """Fraction of the edges whose source lies within window() 16-row blocks
        of the destination's block: what the slab kernel's shared-memory ring
        serves (the rest are far / global loads).  Computed once."""
        if self._ring_cov is None:
            E = self.num_edges
            if E == 0:
                self._ring_cov = 1.0
            else:
                d = (self.col_idx.to(torch.int64) // 16 - self.rows().to(torch.int64) // 16).abs()
                self._ring_cov = float((d <= self.window()).sum().item()) / E
        return self._ring_cov

    def touched(self) -> torch.Tensor:
        """bool[V]: row has >= 1 edge (kernels.py:121)."""
        if self._touched is None:
            # torch.bool is one byte holding 0/1: the kernel writes it as uint8
            t = torch.empty(self.num_vertices, dtype=torch.bool, device=self.row_ptr.device)
            _lib.call("ag_row_touched", self.num_vertices, _lib.ptr(self.row_ptr), _lib.ptr(t),
                      _lib.stream())
            self._touched = t
        return self._touched

    def first_off_block(self, block_size: int) -> int:
        """Index of the first edge crossing a B-block boundary, or -1."""
        if block_size not in self._off_block:
            out = _lib.out_i64()
            _lib.call("ag_first_off_block", self.num_vertices, _lib.ptr(self.row_ptr),
                      _lib.ptr(self.col_idx), int(block_size), _lib.byref(out), _lib.stream())
            self._off_block[block_size] = out.value
        return self._off_block[block_size]

    def role_layout(self, block_size: int):
        """Role-ordered copy of this CSR for the fused kernel, cached per B.

        Every row's edges are re-listed as the intra run (cols in
        [floor(r/B)B, +B), ascending) followed by the inter edges (the row's
        prefix ++ suffix, ascending).  Returns (mid int32[V], col int32[E],
        val f32[E] | None); mid[r] ends row r's intra run.  See
        ag_role_csr_build in include/adaptgear_b200.h.
        """
        if self._long is None:
            self._long = {}
        key = int(block_size)
        lay = self._long.get(key)
        if lay is None:
            dev = self.row_ptr.device
            V, E = self.num_vertices, self.num_edges
            mid = torch.empty(V, dtype=torch.int32, device=dev)
            rcol = torch.empty(E, dtype=torch.int32, device=dev)
            rval = None if self._val is None else torch.empty(E, dtype=torch.float32, device=dev)
            _lib.call("ag_role_csr_build", V, _lib.ptr(self.row_ptr), _lib.ptr(self.col_idx),
                      _lib.ptr(self._val), key, _lib.ptr(rcol), _lib.ptr(rval), _lib.ptr(mid),
                      _lib.stream())
            lay = (mid, rcol, rval)
            self._long[key] = lay
        return lay

    def slab_layout(self, block_size: int = 0):
        """(mid | None, cv, rowinfo, far_cnt, far_src, weighted) for ag_fused_spmm,
        cached per B: the role-ordered layout (block_size > 0) or the plain CSR
        (0), edges as slab-ring (code, weight) pairs for window()."""
        key = int(block_size)
        lay = self._codes.get(key)
        if lay is None:
            if key > 0:
                mid, col, val = self.role_layout(key)
            else:
                mid, col, val = None, self.col_idx, self._val
            cv, rowinfo, far_cnt, far_src = slab_codes(self.num_vertices, self.row_ptr, col, val,
                                                       mid, self.window())
            lay = (mid, cv, rowinfo, far_cnt, far_src, int(val is not None))
            self._codes[key] = lay
        return lay

    def band_layout(self):
        """(rec, rec_off, far_cnt, far_src, window) for ag_band_spmm, cached:
        the inter edges of the B = 16 role layout packed into one record per
        16-row block (ag_band_sizes / ag_band_records), window clipped to the
        band ring's reach."""
        if self._band is None:
            mid, col, val = self.role_layout(16)
            dev = self.row_ptr.device
            V = self.num_vertices
            nb = max((V + 15) // 16, 1)
            sizes = torch.zeros(nb, dtype=torch.int32, device=dev)
            mx = _lib.out_i64()
            _lib.call("ag_band_sizes", V, _lib.ptr(self.row_ptr), _lib.ptr(mid), _lib.ptr(sizes),
                      _lib.byref(mx), _lib.stream())
            off = torch.zeros(nb + 1, dtype=torch.int64, device=dev)
            torch.cumsum(sizes, 0, out=off[1:])
            total = int(off[-1].item())
            if total >= 2 ** 31:
                raise ValueError("band records exceed int32 offsets")
            off = off.to(torch.int32)
            rec = torch.zeros(max(total, 1) * 4, dtype=torch.int32, device=dev)
            cap = int(_lib.load().ag_slab_far_capacity())
            far_cnt = torch.zeros(nb, dtype=torch.int32, device=dev)
            far_src = torch.zeros(nb * cap, dtype=torch.int32, device=dev)
            window = min(self.window(), int(_lib.load().ag_band_max_window()))
            _lib.call("ag_band_records", V, _lib.ptr(self.row_ptr), _lib.ptr(col), _lib.ptr(val),
                      _lib.ptr(mid), window, _lib.ptr(off), _lib.ptr(rec), _lib.ptr(far_cnt),
                      _lib.ptr(far_src), _lib.stream())
            self._band = (rec, off, far_cnt, far_src, window)
        return self._band

    def dense_blocks16(self) -> torch.Tensor:
        """The intra runs of the B = 16 role layout as dense 16 x 16 blocks
        (ag_slab_dense_blocks), cached: the dense-intra fused pair's operand."""
        if self._dense16 is None:
            mid, col, val = self.role_layout(16)
            nb = (self.num_vertices + 15) // 16
            w = torch.empty(max(nb, 1) * 256, dtype=torch.float32, device=self.row_ptr.device)
            _lib.call("ag_slab_dense_blocks", self.num_vertices, _lib.ptr(self.row_ptr),
                      _lib.ptr(mid), _lib.ptr(col), _lib.ptr(val), _lib.ptr(w), _lib.stream())
            self._dense16 = w
        return self._dense16

    def rows(self) -> torch.Tensor:
        """Destination of every edge (the COO row array)."""
        if self._rows is None:
            counts = (self.row_ptr[1:] - self.row_ptr[:-1]).to(torch.int64)
            self._rows = torch.repeat_interleave(
                torch.arange(self.num_vertices, dtype=torch.int32, device=self.row_ptr.device),
                counts)
        return self._rows


class DenseBlockSet:
    """Diagonal B x B blocks of an intra-community adjacency (formats.py:48-73).

    Only communities with >= 1 edge are stored; `comm_slot[c]` maps every
    community to its slot or -1 (device-side lookup for the block kernel).
    """

    __slots__ = ("num_vertices", "block_size", "community_ids", "blocks", "row_touched",
                 "comm_slot", "_panels")

    def __init__(self, num_vertices, block_size, community_ids, blocks, row_touched, comm_slot):
        self.num_vertices = int(num_vertices)
        self.block_size = int(block_size)
        self.community_ids = community_ids
        self.blocks = blocks
        self.row_touched = row_touched
        self.comm_slot = comm_slot
        self._panels = None

    @property
    def panel(self) -> int:
        """Panel width of the tensor-core layout: max(B, 128)."""
        return max(self.block_size, 128)

    def tc_ok(self) -> bool:
        """B divides 128 or is a multiple of 128 (block-diagonal panels)."""
        B = self.block_size
        return (B <= 128 and 128 % B == 0) or B % 128 == 0

    def panels(self) -> torch.Tensor:
        """The blocks as block-diagonal [V, panel] panels (ag_dense_block_pack),
        cached: the A operand of the tensor-core dense_block product."""
        if self._panels is None:
            P = self.panel
            a = torch.empty((self.num_vertices, P), dtype=torch.float32, device=self.blocks.device)
            _lib.call("ag_dense_block_pack", self.num_vertices, self.block_size, P,
                      _lib.ptr(self.comm_slot), _lib.ptr(self.blocks), _lib.ptr(a), P,
                      _lib.stream())
            self._panels = a
        return self._panels

    def nonzero_count(self) -> int:
        return int(torch.count_nonzero(self.blocks).item())


def to_csr(g: Graph) -> CsrMatrix:
    """CSR of a canonical graph (formats.py:76-88); cached on the graph."""
    a = g._cache.get("csr")
    if a is None:
        row_ptr = torch.empty(g.num_vertices + 1, dtype=torch.int32, device=g.dst.device)
        _lib.call("ag_build_row_ptr", g.num_vertices, g.num_edges, _lib.ptr(g.dst),
                  _lib.ptr(row_ptr), _lib.stream())
        a = CsrMatrix(g.num_vertices, row_ptr, g.src, g.weights, rows=g.dst)
        g._cache["csr"] = a
    return a


def to_coo(g) -> CooMatrix:
    """Canonical COO of a graph or of a CSR matrix (formats.py:91-102)."""
    if isinstance(g, CsrMatrix):
        return CooMatrix(g.num_vertices, g.rows(), g.col_idx, g.kernel_val)
    m = g._cache.get("coo")
    if m is None:
        m = CooMatrix(g.num_vertices, g.dst, g.src, g.weights)
        g._cache["coo"] = m
    return m


def to_dense_blocks(g: Graph, block_size: int) -> DenseBlockSet:
    """Pack a block-local (intra) graph into dense B x B blocks (formats.py:105-140)."""
    if block_size < 1:
        raise ValueError("block_size must be >= 1")
    key = ("blocks", int(block_size))
    d = g._cache.get(key)
    if d is not None:
        return d
    b = int(block_size)
    bad = to_csr(g).first_off_block(b)
    if bad >= 0:
        dd = int(g.dst[bad].item())
        ss = int(g.src[bad].item())
        raise ValueError(f"off-diagonal edge (dst={dd}, src={ss}) "
                         f"is not block-local for block_size={b}")
    k = _lib.out_i64()
    _lib.call("ag_blocks_count", g.num_vertices, g.num_edges, _lib.ptr(g.dst), b, _lib.byref(k),
              _lib.stream())
    k = k.value
    dev = g.dst.device
    ncomm = (g.num_vertices + b - 1) // b
    community_ids = torch.empty(k, dtype=torch.int32, device=dev)
    comm_slot = torch.empty(ncomm, dtype=torch.int32, device=dev)
    blocks = torch.empty((k, b, b), dtype=torch.float32, device=dev)
    touched = torch.empty((k, b), dtype=torch.bool, device=dev)
    _lib.call("ag_blocks_fill", g.num_vertices, g.num_edges, _lib.ptr(g.dst), _lib.ptr(g.src),
              _lib.ptr(g.weights), b, k, _lib.ptr(community_ids), _lib.ptr(comm_slot),
              _lib.ptr(blocks), _lib.ptr(touched), _lib.stream())
    d = DenseBlockSet(g.num_vertices, b, community_ids, blocks, touched, comm_slot)
    g._cache[key] = d
    return d


def feature_matrix(data, num_vertices: int | None = None) -> torch.Tensor:
    """Validated C-contiguous fp32 [V, F] device feature matrix."""
    x = as_device(data, torch.float32)
    if x.dim() != 2:
        raise ValueError(f"features must be 2-d, got shape {tuple(x.shape)}")
    if num_vertices is not None and x.shape[0] != num_vertices:
        raise ValueError(f"feature rows {x.shape[0]} != num_vertices {num_vertices}")
    if not bool(torch.isfinite(x).all()):
        raise ValueError("features contain NaN or Inf")
    return x


def random_features(num_vertices: int, dim: int, seed: int = 0) -> torch.Tensor:
    """default_rng(seed).standard_normal((V, F)).astype(f32) (formats.py:158-161)."""
    rng = np.random.default_rng(seed)
    return as_device(rng.standard_normal((num_vertices, dim)).astype(np.float32), torch.float32)
