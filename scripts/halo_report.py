"""Halo volume of the C5 row partition at G = 2/4/8:
rows each rank needs from its peers (= what the per-peer all-to-all moves)
against what the first version's padded all-gather delivered, and how many of
the remote edges read sources near the partition boundary (within the slab
ring's window of the destination block) vs far away.

    python scripts/halo_report.py > profiles/r02_halo_c5.json
"""
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2305_17408_b200 import dist as D  # noqa: E402
from paper_2305_17408_b200.decompose import full_graph  # noqa: E402
from paper_2305_17408_b200.formats import to_csr  # noqa: E402


def main():
    cfg = bench.CONFIGS["C5"]
    _, rg, dec, net, _ = bench.build_workload(cfg)
    out = {"config": "C5", "V": cfg["V"], "edges": rg.num_edges, "partitions": []}
    for name, sub in (("fwd", dec), ("bwd", net.subject_t)):
        csr = to_csr(full_graph(sub))
        H = csr.window()
        V = csr.num_vertices
        counts = (csr.row_ptr[1:] - csr.row_ptr[:-1]).to(torch.int64)
        dst = torch.repeat_interleave(torch.arange(V, device=counts.device), counts)
        src = csr.col_idx.to(torch.int64)
        for G in (2, 4, 8):
            bounds = D.balanced_bounds(csr.row_ptr, G, 16)
            need = D.peer_sets(csr.row_ptr, csr.col_idx, bounds)
            S = D.send_sets(csr.row_ptr, csr.col_idx, bounds)
            allgather = G * max(int(s.numel()) for s in S)
            do, so = D.owner_of(dst, bounds), D.owner_of(src, bounds)
            remote = do != so
            near = remote & ((src // 16 - dst // 16).abs() <= H)
            ranks = []
            for k in range(G):
                need_k = sum(int(need[(k, j)].numel()) for j in range(G) if j != k)
                ranks.append({"rank": k, "rows": bounds[k + 1] - bounds[k], "halo_rows": need_k,
                              "allgather_rows": allgather,
                              "overdelivery_avoided": round(allgather / max(1, need_k), 2)})
            out["partitions"].append({
                "direction": name, "G": G, "window_blocks": H,
                "remote_edge_fraction": round(float(remote.float().mean()), 5),
                "remote_edges_within_window_of_boundary": int(near.sum()),
                "remote_edges_far": int((remote & ~near).sum()),
                "halo_rows_mean_per_rank": round(sum(r["halo_rows"] for r in ranks) / G),
                "halo_rows_over_V": round(sum(r["halo_rows"] for r in ranks) / G / V, 4),
                "allgather_rows_over_V": round(allgather / V, 4),
                "ranks": ranks})
            print(json.dumps(out["partitions"][-1]), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
