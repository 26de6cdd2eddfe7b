"""Full-size host timing of C5 aggregations with the reference's kernels
(oracle/baseline.py), to validate the sampled CPU baseline: one complete
F=100 and one complete F=256 forward aggregation (every row, intra role with
dense_block and with csr_intra_blocked, inter role csr_inter, combine), next
to the V/rows-scaled estimate of the same aggregation from block samples.

    python scripts/cpu_fullscale.py > gpurun_out/cpu_fullscale_c5.json
"""
import json
import os
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import bench  # noqa: E402
from oracle import baseline as B  # noqa: E402


def main():
    cfg = bench.CONFIGS["C5"]
    t0 = time.perf_counter()
    d, s, w = bench._numpy_graph(cfg)
    out = {"config": "C5", "V": cfg["V"], "edges": int(len(d)), "graph_build_numpy_s":
           round(time.perf_counter() - t0, 1), "threads": os.cpu_count(), "runs": []}
    V = cfg["V"]
    rng = np.random.default_rng(0)
    srcs = {f: rng.standard_normal((V, f), dtype=np.float32) for f in (100, 256)}
    for frac in (1.0, 0.015, 0.005):
        ep = B.SampledEpoch(V, d, s, w, 16, cfg["dims"], "gcn", frac=frac, seed=0)
        for f in (100, 256):
            for kind in ("dense_block", "csr_intra_blocked"):
                ep.choice[("fwd", f)] = kind
                tm = {"agg": 0.0}
                ep.aggregate(("fwd", f), srcs[f], tm)
                r = {"frac_rows": round(ep.frac, 5), "F": f, "intra": kind,
                     "wall_s": round(tm["agg"], 2),
                     "full_aggregation_s": round(tm["agg"] * ep.scale, 2)}
                out["runs"].append(r)
                print(json.dumps(r), file=sys.stderr, flush=True)
        ep.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
