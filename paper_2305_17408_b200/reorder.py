"""Community reordering (reference reorder.py:20-228).

cluster_bfs runs the bit-exact host C++ restatement (ag_cluster_bfs: greedy
heap BFS packing + size-preserving swap refinement);
load_partition parses the file here and runs the stable-sort / chunk /
renumber core natively (ag_partition_from_ids); apply_reorder relabels and
re-canonicalises on the device.  Partition arrays are host int64 numpy
arrays, as in the reference.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .graph import Graph, _canonical


@dataclass(frozen=True)
class Partition:
    """Vertex -> community assignment and its old-id -> new-id permutation."""

    num_vertices: int
    community_of: np.ndarray
    permutation: np.ndarray
    comm_size: int

    def __post_init__(self):
        self.community_of.setflags(write=False)
        self.permutation.setflags(write=False)

    @property
    def num_communities(self) -> int:
        return int(self.community_of.max()) + 1 if self.num_vertices else 0


def cluster_bfs(g: Graph, comm_size: int, seed: int = 0) -> Partition:
    """Greedy BFS packing into communities of <= comm_size (reorder.py:92-153).

    Deterministic; ``seed`` is accepted for interface stability only, as in
    the reference.
    """
    del seed
    if comm_size < 1:
        raise ValueError("comm_size must be >= 1")
    n = g.num_vertices
    dst, src, _ = g.numpy()
    dst = np.ascontiguousarray(dst, dtype=np.int32)
    src = np.ascontiguousarray(src, dtype=np.int32)
    comm = np.empty(n, dtype=np.int64)
    perm = np.empty(n, dtype=np.int64)
    _lib.call("ag_cluster_bfs", n, int(dst.size), _lib.host_ptr(dst), _lib.host_ptr(src),
              int(comm_size), _lib.host_ptr(comm), _lib.host_ptr(perm))
    return Partition(num_vertices=n, community_of=comm, permutation=perm, comm_size=comm_size)


def partition_from_ids(ids, comm_size: int) -> Partition:
    """Stable-sort community ids, chunk runs into <= comm_size, renumber."""
    if comm_size < 1:
        raise ValueError("comm_size must be >= 1")
    ids = np.ascontiguousarray(np.asarray(ids, dtype=np.int64))
    n = ids.size
    comm = np.empty(n, dtype=np.int64)
    perm = np.empty(n, dtype=np.int64)
    _lib.call("ag_partition_from_ids", n, _lib.host_ptr(ids), int(comm_size),
              _lib.host_ptr(comm), _lib.host_ptr(perm))
    return Partition(num_vertices=n, community_of=comm, permutation=perm, comm_size=comm_size)


def load_partition(path, comm_size: int) -> Partition:
    """Partition file with one community id per line (reorder.py:156-203)."""
    if comm_size < 1:
        raise ValueError("comm_size must be >= 1")
    raw: list[int] = []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            line = line.strip()
            if not line:
                continue
            try:
                cid = int(line)
            except ValueError:
                raise ValueError(f"{path}:{lineno}: non-integer community id {line!r}")
            if cid < 0:
                raise ValueError(f"{path}:{lineno}: negative community id {cid}")
            raw.append(cid)
    return partition_from_ids(np.array(raw, dtype=np.int64), comm_size)


def identity_partition(num_vertices: int, comm_size: int) -> Partition:
    """No-op reordering: communities are consecutive id ranges."""
    ids = np.arange(num_vertices, dtype=np.int64)
    return Partition(num_vertices=num_vertices, community_of=ids // comm_size,
                     permutation=ids.copy(), comm_size=comm_size)


def apply_reorder(g: Graph, p: Partition) -> Graph:
    """Relabel (perm[dst], perm[src]) and re-canonicalise; weights carry over."""
    if p.num_vertices != g.num_vertices:
        raise ValueError(
            f"partition covers {p.num_vertices} vertices, graph has {g.num_vertices}")
    dev = _lib.device()
    perm = torch.from_numpy(np.array(p.permutation, dtype=np.int64, copy=True)).to(dev)
    E = g.num_edges
    d64 = torch.empty(E, dtype=torch.int64, device=dev)
    s64 = torch.empty(E, dtype=torch.int64, device=dev)
    _lib.call("ag_relabel", E, _lib.ptr(perm), _lib.ptr(g.dst), _lib.ptr(g.src), _lib.ptr(d64),
              _lib.ptr(s64), _lib.stream())
    return _canonical(g.num_vertices, d64, s64, g.weights)
