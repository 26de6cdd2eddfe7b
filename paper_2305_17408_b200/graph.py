"""Device-resident canonical graphs (reference graph.py:28-106).

A Graph holds its canonical (dst, src) edge set as int32 CUDA tensors sorted
by key dst*V+src with duplicates merged (fp64-summed weights rounded to fp32),
exactly as Graph.from_edges does (graph.py:47-82); the canonicalisation runs
on the device (ag_canonicalize: radix sort + unique + segmented fp64 sum).
Derived device data (in-degrees, CSR, ...) is cached on the instance, which is
immutable by contract like the reference's read-only arrays.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import EdgeListError

MAX_VERTICES = 2**31 - 1


def as_device(a, dtype: torch.dtype) -> torch.Tensor:
    """Contiguous CUDA tensor of `dtype` from a tensor / ndarray / sequence."""
    dev = _lib.device()
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    np_dtype = {torch.int64: np.int64, torch.int32: np.int32, torch.float32: np.float32}[dtype]
    arr = np.ascontiguousarray(np.asarray(a, dtype=np_dtype))
    if not arr.flags.writeable:  # read-only host input (the reference's arrays are)
        return torch.tensor(arr, device=dev)
    return torch.from_numpy(arr).to(dev)


@dataclass(frozen=True)
class Graph:
    """Directed graph as a canonical (dst, src) edge set on the device."""

    num_vertices: int
    dst: torch.Tensor
    src: torch.Tensor
    weights: torch.Tensor | None = None
    _cache: dict = field(default_factory=dict, compare=False, repr=False)

    @classmethod
    def from_edges(cls, num_vertices, dst, src, weights=None) -> "Graph":
        """Canonical graph from raw edges: sort, dedup, fp64-merge weights."""
        if num_vertices < 0 or num_vertices > MAX_VERTICES:
            raise ValueError(f"invalid vertex count {num_vertices}")
        d = as_device(dst, torch.int64)
        s = as_device(src, torch.int64)
        if d.shape != s.shape or d.dim() != 1:
            raise ValueError("dst and src must be 1-d arrays of equal length")
        w = None
        if weights is not None:
            w = as_device(weights, torch.float32)
            if w.shape != d.shape:
                raise ValueError("weights must have one entry per edge")
        return _canonical(int(num_vertices), d, s, w)

    @property
    def num_edges(self) -> int:
        return int(self.dst.numel())

    def edge_weights(self) -> torch.Tensor:
        """Per-edge weights; implicit 1.0 when the graph is unweighted."""
        if self.weights is not None:
            return self.weights
        w = self._cache.get("ones")
        if w is None:
            w = torch.ones(self.num_edges, dtype=torch.float32, device=self.dst.device)
            self._cache["ones"] = w
        return w

    def in_degrees(self) -> torch.Tensor:
        """int64 in-degree per vertex (row counts of A)."""
        deg = self._cache.get("in_deg")
        if deg is None:
            deg = torch.empty(self.num_vertices, dtype=torch.int64, device=self.dst.device)
            _lib.call("ag_in_degrees", self.num_vertices, self.num_edges, _lib.ptr(self.dst),
                      _lib.ptr(deg), _lib.stream())
            self._cache["in_deg"] = deg
        return deg

    def out_degrees(self) -> torch.Tensor:
        deg = torch.empty(self.num_vertices, dtype=torch.int64, device=self.dst.device)
        _lib.call("ag_in_degrees", self.num_vertices, self.num_edges, _lib.ptr(self.src),
                  _lib.ptr(deg), _lib.stream())
        return deg

    def reverse(self) -> "Graph":
        """Edge-reversed graph (transpose of the adjacency matrix), cached."""
        r = self._cache.get("reverse")
        if r is None:
            r = _canonical(self.num_vertices, self.src.to(torch.int64), self.dst.to(torch.int64),
                           self.weights)
            self._cache["reverse"] = r
        return r

    def edge_set(self) -> set[tuple[int, int]]:
        return set(zip(self.dst.cpu().tolist(), self.src.cpu().tolist()))

    def numpy(self):
        """(dst, src, weights|None) as host numpy arrays."""
        w = None if self.weights is None else self.weights.cpu().numpy()
        return self.dst.cpu().numpy(), self.src.cpu().numpy(), w


def _canonical(V: int, d: torch.Tensor, s: torch.Tensor, w: torch.Tensor | None) -> Graph:
    E = int(d.numel())
    dev = _lib.device()
    dst_out = torch.empty(E, dtype=torch.int32, device=dev)
    src_out = torch.empty(E, dtype=torch.int32, device=dev)
    w_out = torch.empty(E, dtype=torch.float32, device=dev) if w is not None else None
    nu = _lib.out_i64()
    _lib.call("ag_canonicalize", V, E, _lib.ptr(d), _lib.ptr(s), _lib.ptr(w), _lib.ptr(dst_out),
              _lib.ptr(src_out), _lib.ptr(w_out), _lib.byref(nu), _lib.stream())
    n = nu.value
    if n != E:
        dst_out, src_out = dst_out[:n].clone(), src_out[:n].clone()
        if w_out is not None:
            w_out = w_out[:n].clone()
    return Graph(num_vertices=V, dst=dst_out, src=src_out, weights=w_out)


def load_edge_list(path, weighted: bool = False) -> Graph:
    """Plain-text edge list, "src dst [weight]" per line (graph.py:109-160).

    '#' lines are comments; an optional "% vertices N" header fixes V,
    otherwise V = 1 + the largest id.  Errors name the file and line.
    """
    dsts: list[int] = []
    srcs: list[int] = []
    wts: list[float] = []
    header = None
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            line = raw.strip()
            if not line or line.startswith("#"):
                continue
            if line.startswith("%"):
                parts = line[1:].split()
                if len(parts) == 2 and parts[0] == "vertices":
                    try:
                        header = int(parts[1])
                    except ValueError:
                        raise EdgeListError(f"{path}:{lineno}: bad vertex header {line!r}")
                continue
            parts = line.split()
            need = 3 if weighted else 2
            if len(parts) < need:
                want = "src dst weight" if weighted else "src dst"
                raise EdgeListError(f"{path}:{lineno}: expected {want}, got {line!r}")
            try:
                s, d = int(parts[0]), int(parts[1])
            except ValueError:
                raise EdgeListError(f"{path}:{lineno}: non-integer vertex id in {line!r}")
            if s < 0 or d < 0:
                raise EdgeListError(f"{path}:{lineno}: negative vertex id in {line!r}")
            if s > MAX_VERTICES or d > MAX_VERTICES:
                raise EdgeListError(f"{path}:{lineno}: vertex id exceeds 32-bit range")
            if weighted:
                try:
                    wts.append(float(parts[2]))
                except ValueError:
                    raise EdgeListError(f"{path}:{lineno}: non-numeric weight in {line!r}")
            srcs.append(s)
            dsts.append(d)
    if not dsts:
        raise EdgeListError(f"{path}: no edges found")
    V = header if header is not None else 1 + max(max(dsts), max(srcs))
    return Graph.from_edges(V, dsts, srcs, wts if weighted else None)


def replace(g: Graph, **kw) -> Graph:
    return dataclasses.replace(g, _cache={}, **kw)
