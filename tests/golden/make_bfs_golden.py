"""Golden cluster_bfs results at BASELINE config scale (C2 pubmed-shaped,
C3 ogbn-arxiv-shaped) from the UNMODIFIED reference.

Run in the build container (the reference is not on the GPU box):

    python tests/golden/make_bfs_golden.py

The graphs come from oracle/synth.py (the numpy twin of the device
generator, deterministic on any host); the reference's Graph.from_edges and
cluster_bfs (reorder.py:92-153) partition them, and only sha256 digests of
the (community, perm) arrays are stored (tests/golden/bfs_scale.json), so the
fixture stays small.  tests/test_oracle.py checks the host C++ cluster_bfs of
the product (and the oracle restatement) against them.
"""
from __future__ import annotations

import hashlib
import json
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[2]
REF = pathlib.Path("/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(REF))

import adaptgear as ref  # noqa: E402

from oracle import synth  # noqa: E402

# (name, V, E, generator parameters, comm_size): the bench's generator at C2 / C3 size
CASES = [("C2", 19717, 88648, dict(block_gen=16, p_intra=0.4, p_global=0.05, window=16), 16),
         ("C3", 169343, 1166243, dict(block_gen=16, p_intra=0.4, p_global=0.05, window=16), 16)]


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def main():
    out = {"source": "reference adaptgear.reorder.cluster_bfs on oracle.synth.community_graph "
                     "(seed 0); digests are sha256 of int64 arrays", "cases": []}
    for name, V, E, gen, B in CASES:
        (dst, src), _ = synth.community_graph(V, E, seed=0, **gen)
        t0 = time.perf_counter()
        g = ref.Graph.from_edges(V, dst, src)
        part = ref.cluster_bfs(g, B)
        dt = time.perf_counter() - t0
        comm = np.asarray(part.community_of)
        perm = np.asarray(part.permutation)
        out["cases"].append({"name": name, "V": V, "E": E, "generator": gen, "comm_size": B,
                             "edges_canonical": int(np.asarray(g.dst).size),
                             "community_sha256": digest(comm), "perm_sha256": digest(perm),
                             "reference_seconds": round(dt, 1)})
        print(out["cases"][-1], flush=True)
    (pathlib.Path(__file__).resolve().parent / "bfs_scale.json").write_text(
        json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
