"""Generate tests/golden/harness.json from the UNMODIFIED reference harness.

Run in the build container (the reference is not on the GPU box):

    python tests/golden/make_harness_golden.py

Records, for seeded configurations: the RMAT / planted-partition edge sets
(as a digest plus the first keys), the full `run_density` report minus its
wall-clock timings, and the `run_pipeline` report fields that do not depend on
timing (config, density, topology bytes, profiling iterations, locked pair for
O1, result checksum).  Pins paper_2305_17408_b200.generators /
pipeline.build_graph (CPU, tests/test_harness.py) and paper_2305_17408_b200.harness
(GPU).
"""
from __future__ import annotations

import hashlib
import json
import pathlib
import sys

import numpy as np

REF = pathlib.Path("/root/reference/pkg/src")
OUT = pathlib.Path(__file__).resolve().parent / "harness.json"
sys.path.insert(0, str(REF))

from adaptgear import bench as rb  # noqa: E402
from adaptgear import graph as rg  # noqa: E402

RMAT_CASES = [  # (V, E, probs, seed)
    (100, 500, rg.RMAT_DEFAULT_PROBS, 0),
    (1, 1, rg.RMAT_DEFAULT_PROBS, 0),
    (37, 1369, rg.RMAT_DEFAULT_PROBS, 3),
    (64, 3000, (0.9, 0.05, 0.05, 0.0), 1),  # unreachable cells: complement fill
    (2048, 1 << 14, (0.25, 0.25, 0.25, 0.25), 0),
    (5000, 60000, rg.RMAT_DEFAULT_PROBS, 7),
]
PLANTED_CASES = [  # (groups, size, p_in, p_out, seed, shuffle)
    (8, 16, 0.5, 0.01, 0, True),
    (4, 16, 0.4, 0.02, 2, True),
    (5, 7, 0.6, 0.05, 1, False),
]
DENSITY_CASES = [
    dict(),
    dict(rmat=(300, 3000), reorder="none"),
    dict(rmat=(300, 3000), reorder="bfs", comm_size=8),
    dict(planted=(6, 16, 0.4, 0.02), model="gcn"),
]
PIPELINE_CASES = [
    dict(mode=m, model=model, op=op, iters=8, profile_iters=1, feat_dim=16)
    for m in ("O1", "O2", "O3")
    for model, op in (("agg_only", "sum"), ("agg_only", "mean"), ("agg_only", "max"),
                      ("gcn", "sum"), ("gin", "sum"))
    if not (m == "O2" and op == "max")
] + [dict(mode="O3", rmat=(400, 5000), feat_dim=24, iters=6, profile_iters=1)]


def digest(keys: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(keys, dtype=np.int64).tobytes()).hexdigest()


def main():
    out = {"numpy": np.__version__, "reference": str(REF), "rmat": [], "planted": [],
           "density": [], "pipeline": []}
    for v, e, probs, seed in RMAT_CASES:
        g = rg.generate_rmat(v, e, probs=probs, seed=seed)
        keys = g.dst.astype(np.int64) * v + g.src
        out["rmat"].append({"V": v, "E": e, "probs": list(probs), "seed": seed,
                            "sha256": digest(keys), "head": keys[:16].tolist()})
    for groups, size, p_in, p_out, seed, shuffle in PLANTED_CASES:
        g, labels = rg.generate_planted_partition(groups, size, p_in, p_out, seed=seed,
                                                  shuffle=shuffle)
        n = groups * size
        keys = g.dst.astype(np.int64) * n + g.src
        out["planted"].append({"groups": groups, "size": size, "p_in": p_in, "p_out": p_out,
                               "seed": seed, "shuffle": shuffle, "num_edges": int(keys.size),
                               "sha256": digest(keys), "labels": labels.tolist()})
    for kw in DENSITY_CASES:
        rep = rb.run_density(rb.RunConfig(**kw))
        rep.pop("preprocessing_ms")
        out["density"].append({"kwargs": {k: list(v) if isinstance(v, tuple) else v
                                          for k, v in kw.items()}, "report": rep})
    for kw in PIPELINE_CASES:
        rep = rb.run_pipeline(rb.RunConfig(**kw))
        keep = {k: rep[k] for k in ("config", "density", "topology_bytes", "locked")}
        keep["profiling_iters"] = rep["totals"]["profiling_iters"]
        keep["result_checksum"] = rep["totals"]["result_checksum"]
        keep["num_iterations"] = len(rep["iterations"])
        if kw["mode"] != "O1":
            keep.pop("locked")  # timing-dependent
        out["pipeline"].append({"kwargs": {k: list(v) if isinstance(v, tuple) else v
                                           for k, v in kw.items()}, "report": keep})
    OUT.write_text(json.dumps(out, indent=1) + "\n")
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
