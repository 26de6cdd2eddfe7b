"""Synthetic graph sources of the reference harness (graph.py:163-259):
`generate_rmat` and `generate_planted_partition`.

Sampling stays on the host with the reference's numpy RNG stream, draw for
draw, so a seed yields the same edge set as the reference (pinned by
tests/golden/harness.json); only canonicalisation (`Graph.from_edges`) runs on
the device.  `rmat_keys` / `planted_edges` are the host halves, importable
without a GPU.  Neither scales to the benchmark shapes (planted partition
draws an n x n mask): those come from `synth.community_graph`.
"""
from __future__ import annotations

import numpy as np

RMAT_DEFAULT_PROBS = (0.57, 0.19, 0.19, 0.05)
_COMPLEMENT_CAP = 1 << 27  # cells; past this a stalled sampler cannot fill from the complement
_STALL_LIMIT = 50


def _next_power_of_two(n: int) -> int:
    return 1 if n <= 1 else 1 << (int(n) - 1).bit_length()


def rmat_keys(num_vertices: int, num_edges: int, probs=RMAT_DEFAULT_PROBS,
              seed: int = 0) -> np.ndarray:
    """Sorted distinct edge keys dst*V+src of an RMAT graph (graph.py:167-227).

    The recursion runs on the next power of two >= V; samples outside the
    range are discarded; batches of max(4*need, 1024) draws of `levels`
    uniforms each are merged with np.unique and truncated to `num_edges`; 50
    batches without a new key fall back to a uniform fill from the complement.
    """
    if num_vertices <= 0:
        raise ValueError("num_vertices must be positive")
    a, b, c, d = (float(p) for p in probs)
    if min(a, b, c, d) < 0 or abs(a + b + c + d - 1.0) > 1e-9:
        raise ValueError(f"quadrant probabilities must be >= 0 and sum to 1, got {probs}")
    cells = num_vertices * num_vertices
    if num_edges < 0 or num_edges > cells:
        raise ValueError(f"cannot place {num_edges} distinct edges in "
                         f"{num_vertices}x{num_vertices} cells")
    rng = np.random.default_rng(seed)
    if num_edges == cells:
        return np.arange(cells, dtype=np.int64)
    levels = _next_power_of_two(num_vertices).bit_length() - 1
    cuts = np.array([a, a + b, a + b + c])
    weights = (np.int64(1) << np.arange(levels - 1, -1, -1, dtype=np.int64)) if levels else None
    keys = np.empty(0, dtype=np.int64)
    stalls = 0
    while keys.size < num_edges:
        batch = max(4 * (num_edges - keys.size), 1024)
        if levels == 0:
            cand = np.zeros(batch, dtype=np.int64)
        else:
            quad = np.digitize(rng.random((batch, levels)), cuts)
            dst = (quad >> 1).astype(np.int64) @ weights
            src = (quad & 1).astype(np.int64) @ weights
            ok = (dst < num_vertices) & (src < num_vertices)
            cand = dst[ok] * num_vertices + src[ok]
        merged = np.unique(np.concatenate([keys, cand]))
        stalls = stalls + 1 if merged.size == keys.size else 0
        keys = merged[:num_edges]
        if stalls >= _STALL_LIMIT:
            if cells > _COMPLEMENT_CAP:
                raise ValueError("RMAT sampling stalled and the cell space is "
                                 "too large for complement filling")
            rest = np.setdiff1d(np.arange(cells, dtype=np.int64), keys)
            extra = rng.choice(rest, size=num_edges - keys.size, replace=False)
            keys = np.sort(np.concatenate([keys, extra]))
            break
    return keys


def planted_edges(num_groups: int, group_size: int, p_in: float, p_out: float,
                  seed: int = 0, shuffle: bool = True):
    """(dst, src, labels) of a directed planted-partition graph (graph.py:230-259):
    each ordered pair u != v is an edge with probability p_in inside a group,
    p_out across; `shuffle` permutes the vertex ids."""
    if num_groups < 1 or group_size < 1:
        raise ValueError("num_groups and group_size must be >= 1")
    n = num_groups * group_size
    rng = np.random.default_rng(seed)
    groups = np.repeat(np.arange(num_groups), group_size)
    same = groups[:, None] == groups[None, :]
    mask = rng.random((n, n)) < np.where(same, p_in, p_out)
    np.fill_diagonal(mask, False)
    dst, src = np.nonzero(mask)
    if not shuffle:
        return dst, src, groups.astype(np.int64)
    id_map = rng.permutation(n)
    labels = np.empty(n, dtype=np.int64)
    labels[id_map] = groups
    return id_map[dst], id_map[src], labels


def generate_rmat(num_vertices: int, num_edges: int, probs=RMAT_DEFAULT_PROBS, seed: int = 0):
    from .graph import Graph
    keys = rmat_keys(num_vertices, num_edges, probs, seed)
    return Graph.from_edges(num_vertices, keys // num_vertices, keys % num_vertices)


def generate_planted_partition(num_groups: int, group_size: int, p_in: float, p_out: float,
                               seed: int = 0, shuffle: bool = True):
    from .graph import Graph
    dst, src, labels = planted_edges(num_groups, group_size, p_in, p_out, seed, shuffle)
    return Graph.from_edges(num_groups * group_size, dst, src), labels
