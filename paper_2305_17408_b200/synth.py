"""Seeded O(E) community-graph generator.

The reference generators cannot build the C3-C5 configurations
(generate_planted_partition draws a dense V x V mask, graph.py:246-248;
generate_rmat draws 4E x levels doubles, graph.py:202-206).  This generator
is a pure function of (parameters, candidate index): candidate i is decoded
on the device from splitmix64 hashes by `ag_synth_candidates`, so the numpy
restatement in oracle/synth.py produces the identical graph at test sizes.

Candidate i (pre-shuffle ids, communities of `block_gen` consecutive ids):
  dst   = floor(V * u0^skew)                      (skew=1: uniform)
  intra with probability p_intra: a different member of dst's community
  inter otherwise: with probability p_global a uniform community, else the
        community at offset +-(1 + floor(u4 * window)) (locality), then a
        uniform member; self loops are dropped.
The first E distinct (dst, src) keys in candidate order are kept (exactly E
edges, like graph.py:200-216), then ids are shuffled by the rank of a 64-bit
vertex hash and the graph is canonicalised.  `communities[v]` is the planted
community of (shuffled) vertex v, i.e. a METIS-style partition file.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .graph import Graph

SIGN = -(2**63)


def candidates(V: int, block_gen: int, p_intra: float, p_global: float, window: int,
               skew: int, seed: int, first: int, count: int):
    dev = _lib.device()
    d = torch.empty(count, dtype=torch.int64, device=dev)
    s = torch.empty(count, dtype=torch.int64, device=dev)
    _lib.call("ag_synth_candidates", V, block_gen, float(p_intra), float(p_global), window, skew,
              seed & 0xFFFFFFFFFFFFFFFF, first, count, _lib.ptr(d), _lib.ptr(s), _lib.stream())
    return d, s


def vertex_permutation(V: int, seed: int) -> torch.Tensor:
    """perm[v] = rank of hash(seed, v) (ties impossible in 64 bits; stable anyway)."""
    dev = _lib.device()
    keys = torch.empty(V, dtype=torch.int64, device=dev)
    _lib.call("ag_synth_vertex_keys", V, seed & 0xFFFFFFFFFFFFFFFF, _lib.ptr(keys), _lib.stream())
    order = torch.argsort(keys ^ SIGN, stable=True)  # unsigned order
    perm = torch.empty(V, dtype=torch.int64, device=dev)
    perm[order] = torch.arange(V, dtype=torch.int64, device=dev)
    return perm


def community_graph(V: int, E: int, block_gen: int = 16, p_intra: float = 0.5,
                    p_global: float = 0.1, window: int = 4, skew: int = 1, seed: int = 0):
    """Returns (Graph, communities int64[V] host array)."""
    if E > V * (V - 1):
        raise ValueError(f"cannot place {E} distinct edges without self loops on {V} vertices")
    n = E + E // 16 + 1024
    while True:
        d, s = candidates(V, block_gen, p_intra, p_global, window, skew, seed, 0, n)
        idx = torch.arange(n, dtype=torch.int64, device=d.device)
        ok = s >= 0
        keys = d[ok] * V + s[ok]
        idx = idx[ok]
        uniq, inv = torch.unique(keys, return_inverse=True)
        if uniq.numel() >= E:
            break
        n += 2 * (E - uniq.numel()) + 1024
    first = torch.full((uniq.numel(),), n, dtype=torch.int64, device=d.device)
    first.scatter_reduce_(0, inv, idx, reduce="amin")
    chosen = uniq[torch.argsort(first, stable=True)[:E]]
    del d, s, keys, idx, inv, first, uniq
    perm = vertex_permutation(V, seed)
    dst = perm[chosen // V]
    src = perm[chosen % V]
    g = Graph.from_edges(V, dst, src)
    comm = torch.empty(V, dtype=torch.int64, device=perm.device)
    comm[perm] = torch.arange(V, dtype=torch.int64, device=perm.device) // block_gen
    return g, comm.cpu().numpy()


def labels_and_mask(V: int, num_classes: int, seed: int = 0):
    """Seeded labels and a ~50% train mask, host numpy."""
    rng = np.random.default_rng(seed + 7919)
    labels = rng.integers(0, num_classes, V).astype(np.int32)
    mask = rng.random(V) < 0.5
    return labels, mask
