"""Generate the golden vectors of tests/golden/ from the UNMODIFIED reference.

Run in the build container (the reference is not on the GPU box):

    python tests/golden/make_golden.py

It imports `adaptgear` read-only from /root/reference/pkg/src (numpy only; the
matplotlib-dependent cli/plots modules are never imported) and records the
reference's outputs on seeded inputs.  The fixtures pin the oracle
(tests/test_oracle.py, CPU) and the device path (tests/test_parity_gpu.py).
"""
from __future__ import annotations

import json
import pathlib
import sys

import numpy as np

REF = pathlib.Path("/root/reference/pkg/src")
OUT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

import adaptgear as ag  # noqa: E402
from adaptgear import AggregateOp  # noqa: E402

OPS = (AggregateOp.SUM, AggregateOp.MEAN, AggregateOp.MAX)


def raw_graph(rng, V, density, weighted, dup_frac=0.1):
    """Random raw edge arrays WITH duplicates (exercises from_edges merging)."""
    E = max(1, int(density * V * V))
    keys = rng.choice(V * V, size=E, replace=False)
    ndup = int(dup_frac * E)
    if ndup:
        keys = np.concatenate([keys, rng.choice(keys, size=ndup)])
        rng.shuffle(keys)
    dst, src = keys // V, keys % V
    w = rng.uniform(0.1, 2.0, size=keys.size).astype(np.float32) if weighted else None
    return dst.astype(np.int64), src.astype(np.int64), w


def kernel_cases(rng):
    cases = []
    specs = [
        # (V, density, weighted, B, F)
        (3, 0.5, True, 2, 1), (17, 0.3, True, 4, 6), (64, 0.06, False, 16, 8),
        (128, 0.05, True, 16, 32), (200, 0.02, True, 7, 13), (256, 0.1, False, 32, 40),
        (300, 0.01, True, 16, 20), (40, 0.2, True, 16, 256), (24, 0.2, True, 8, 602),
        (12, 0.5, False, 5, 1433), (256, 0.2, False, 16, 4), (21, 0.3, True, 8, 2),
    ]
    for V, dens, weighted, B, F in specs:
        cases.append((V, *raw_graph(rng, V, dens, weighted), B, F))
    # high-degree rows: pairwise recursion depths 1..4
    V = 4096
    rows, cols = [], []
    for r, deg in ((5, 3000), (17, 1000), (300, 129), (301, 128), (302, 257), (4000, 4096)):
        cols.append(rng.choice(V, size=deg, replace=False))
        rows.append(np.full(deg, r))
    dst, src = np.concatenate(rows), np.concatenate(cols)
    w = rng.uniform(0.1, 2.0, size=dst.size).astype(np.float32)
    cases.append((V, dst, src, w, 64, 2))
    cases.append((V, dst, src, None, 64, 1))
    return cases


def main():
    rng = np.random.default_rng(20260517)
    out = {}
    meta = {"numpy": np.__version__, "reference": str(REF), "cases": []}
    for i, (V, d, s, w, B, F) in enumerate(kernel_cases(rng)):
        p = f"k{i}_"
        out[p + "V"] = np.array(V)
        out[p + "B"] = np.array(B)
        out[p + "raw_dst"], out[p + "raw_src"] = d, s
        if w is not None:
            out[p + "raw_w"] = w
        g = ag.Graph.from_edges(V, d, s, w)
        out[p + "dst"], out[p + "src"] = g.dst, g.src
        if w is not None:
            out[p + "w"] = g.weights
        x = rng.standard_normal((V, F)).astype(np.float32)
        out[p + "x"] = x
        a = ag.to_csr(g)
        out[p + "row_ptr"] = a.row_ptr
        dec = ag.decompose(g, B)
        for role, sub in (("intra", dec.intra), ("inter", dec.inter)):
            out[p + role + "_dst"], out[p + role + "_src"] = sub.dst, sub.src
            if sub.weights is not None:
                out[p + role + "_w"] = sub.weights
        out[p + "full_in_degree"] = dec.full_in_degree
        blk = ag.to_dense_blocks(dec.intra, B)
        out[p + "blk_ids"], out[p + "blk_blocks"] = blk.community_ids, blk.blocks
        out[p + "blk_touched"] = blk.row_touched
        icsr = ag.to_csr(dec.intra)
        for op in OPS:
            o = op.value
            pr = ag.aggregate_csr_inter(a, x, op)
            out[p + f"csr_{o}"], out[p + f"csr_{o}_touched"] = pr.values, pr.touched
            out[p + f"intra_{o}"] = ag.aggregate_csr_intra_blocked(icsr, x, op, B).values
            out[p + f"coo_{o}"] = ag.aggregate_coo_atomic(ag.to_coo(g), x, op).values
            out[p + f"full_{o}"] = ag.aggregate_full(g, x, op)
            if op is not AggregateOp.MAX:
                out[p + f"dense_{o}"] = ag.aggregate_dense_block(blk, x, op).values
            for ki in (ag.KernelKind.CSR_INTRA_BLOCKED, ag.KernelKind.DENSE_BLOCK):
                if op is AggregateOp.MAX and ki is ag.KernelKind.DENSE_BLOCK:
                    continue
                for ke in (ag.KernelKind.CSR_INTER, ag.KernelKind.COO_ATOMIC):
                    out[p + f"dec_{o}_{ki.value}_{ke.value}"] = ag.aggregate_decomposed(
                        dec, x, op, kernel_intra=ki, kernel_inter=ke)
            if V <= 4096:
                out[p + f"dref_{o}"] = ag.aggregate_dense_reference(g, x, op)
        out[p + "bwd"] = ag.backward_sum(g.reverse(), x)
        rg = g.reverse()
        out[p + "rev_dst"], out[p + "rev_src"] = rg.dst, rg.src
        gn = ag.gcn_normalize(g)
        out[p + "gcn_dst"], out[p + "gcn_src"], out[p + "gcn_w"] = gn.dst, gn.src, gn.weights
        meta["cases"].append({"V": V, "E": int(g.num_edges), "B": B, "F": F,
                              "weighted": w is not None})
    np.savez_compressed(OUT / "kernels.npz", **out)

    # ------------------------------------------------------------ reorder --
    rout = {}
    specs = []
    for j in range(24):
        V = int(rng.integers(2, 301))
        specs.append(("rand", V, float(rng.uniform(0.002, 0.1)), bool(j % 2),
                      int(rng.integers(1, 33))))
    for j in range(6):
        specs.append(("planted", 16, 0.5, bool(j % 2), 16))
    specs.append(("rand", 3000, 0.002, True, 16))
    specs.append(("planted", 32, 0.4, True, 16))
    for i, (kind, V, dens, gcn, B) in enumerate(specs):
        p = f"r{i}_"
        if kind == "rand":
            d, s, _ = raw_graph(rng, V, dens, False, dup_frac=0.0)
            g = ag.Graph.from_edges(V, d, s)
        else:
            g, _ = ag.generate_planted_partition(V if V < 30 else 8, 16 if V < 30 else 32,
                                                 dens, 0.01, seed=i)
        if gcn:
            g = ag.gcn_normalize(g)
        part = ag.cluster_bfs(g, B)
        rg = ag.apply_reorder(g, part)
        rout[p + "V"], rout[p + "B"] = np.array(g.num_vertices), np.array(B)
        rout[p + "dst"], rout[p + "src"] = g.dst, g.src
        if g.weights is not None:
            rout[p + "w"] = g.weights
        rout[p + "community"], rout[p + "perm"] = part.community_of, part.permutation
        rout[p + "re_dst"], rout[p + "re_src"] = rg.dst, rg.src
        if rg.weights is not None:
            rout[p + "re_w"] = rg.weights
    # load_partition cores (written through a temp file like the reference)
    import tempfile
    for i, (n, hi, B) in enumerate(((5, 1, 2), (100, 7, 4), (1000, 50, 16), (64, 1, 100))):
        ids = rng.integers(0, hi + 1, n)
        with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False) as fh:
            fh.write("\n".join(map(str, ids.tolist())) + "\n")
        part = ag.load_partition(fh.name, B)
        rout[f"lp{i}_ids"], rout[f"lp{i}_B"] = ids, np.array(B)
        rout[f"lp{i}_community"], rout[f"lp{i}_perm"] = part.community_of, part.permutation
    np.savez_compressed(OUT / "reorder.npz", **rout)

    # --------------------------------------------------------- layers -------
    lout = {}
    for i, (model, V, B, fin, fout) in enumerate((("gcn", 64, 16, 8, 4), ("gin", 64, 16, 8, 4),
                                                  ("gcn", 200, 8, 32, 16), ("gin", 150, 16, 5, 7))):
        p = f"l{i}_"
        d, s, _ = raw_graph(rng, V, 0.06, False, dup_frac=0.0)
        g = ag.Graph.from_edges(V, d, s)
        if model == "gcn":
            g = ag.gcn_normalize(g)
        part = ag.cluster_bfs(g, B)
        dec = ag.decompose(ag.apply_reorder(g, part), B)
        x = rng.standard_normal((V, fin)).astype(np.float32)
        xp = np.empty_like(x)
        xp[part.permutation] = x
        params = ag.LayerParams.seeded(model, fin, fout, seed=i, gin_eps=0.2)
        fwd = ag.gcn_layer_forward if model == "gcn" else ag.gin_layer_forward
        lout[p + "model"] = np.array(model)
        lout[p + "V"], lout[p + "B"] = np.array(V), np.array(B)
        lout[p + "dst"], lout[p + "src"] = g.dst, g.src
        if g.weights is not None:
            lout[p + "w"] = g.weights
        lout[p + "perm"] = part.permutation
        lout[p + "x"], lout[p + "weight"] = x, params.weight
        lout[p + "out_decomposed"] = fwd(dec, xp, params)
        lout[p + "out_full"] = fwd(g, x, params)
    # criterion-10 style pipeline golden (the file the reference does not ship)
    g, _ = ag.generate_planted_partition(4, 16, 0.5, 0.02, seed=7)
    x = np.random.default_rng(7).standard_normal((64, 8)).astype(np.float32)
    p_gcn = ag.LayerParams.seeded("gcn", 8, 8, seed=11)
    p_gin = ag.LayerParams.seeded("gin", 8, 8, seed=11, gin_eps=0.1)
    gn = ag.gcn_normalize(g)
    lout["pipe_dst"], lout["pipe_src"] = g.dst, g.src
    lout["pipe_x"] = x
    lout["pipe_gcn"] = ag.gcn_layer_forward(gn, x, p_gcn)
    lout["pipe_gin"] = ag.gin_layer_forward(g, x, p_gin)
    np.savez_compressed(OUT / "layers.npz", **lout)
    (OUT / "meta.json").write_text(json.dumps(meta, indent=1))
    for f in ("kernels.npz", "reorder.npz", "layers.npz"):
        print(f, (OUT / f).stat().st_size)


if __name__ == "__main__":
    main()
