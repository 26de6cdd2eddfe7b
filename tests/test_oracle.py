"""CPU: pin the oracle (oracle/) against the reference's golden vectors.

The goldens were produced by the unmodified reference (tests/golden/make_golden.py);
every integer array must match exactly, every float array bitwise (the
oracle uses the same numpy reductions as the reference).
"""
import numpy as np
import pytest

from conftest import same_float
from oracle import build as obuild
from oracle import ref_numpy as R
from oracle import synth as osynth

OPS = ("sum", "mean", "max")


def graph(z, p, role=""):
    pre = p + (role + "_" if role else "")
    return z[pre + "dst"], z[pre + "src"], z.get(pre + "w")


def test_canonical_and_formats(kernels_golden):
    z = kernels_golden
    for i in z.cases("k"):
        p = f"k{i}_"
        V = int(z[p + "V"])
        d, s, w = R.canonical(V, z[p + "raw_dst"], z[p + "raw_src"], z.get(p + "raw_w"))
        assert np.array_equal(d, z[p + "dst"]) and np.array_equal(s, z[p + "src"])
        if w is not None:
            assert same_float(w, z[p + "w"])
        rp, _, _ = R.to_csr(V, d, s, w)
        assert np.array_equal(rp, z[p + "row_ptr"])
        gd, gs, gw = R.gcn_normalize(V, d, s)
        assert np.array_equal(gd, z[p + "gcn_dst"]) and np.array_equal(gs, z[p + "gcn_src"])
        assert same_float(gw, z[p + "gcn_w"])
        rd, rs, _ = R.canonical(V, s, d, w)
        assert np.array_equal(rd, z[p + "rev_dst"]) and np.array_equal(rs, z[p + "rev_src"])


def test_decompose_and_blocks(kernels_golden):
    z = kernels_golden
    for i in z.cases("k"):
        p = f"k{i}_"
        V, B = int(z[p + "V"]), int(z[p + "B"])
        intra, inter, deg = R.decompose(V, *graph(z, p), B)
        for role, sub in (("intra", intra), ("inter", inter)):
            assert np.array_equal(sub[0], z[p + role + "_dst"])
            assert np.array_equal(sub[1], z[p + role + "_src"])
        assert np.array_equal(deg, z[p + "full_in_degree"])
        ids, blocks, touched = R.to_blocks(V, *intra, B)
        assert np.array_equal(ids, z[p + "blk_ids"])
        assert same_float(blocks, z[p + "blk_blocks"])
        assert np.array_equal(touched, z[p + "blk_touched"])


def test_kernels_bitwise(kernels_golden):
    z = kernels_golden
    for i in z.cases("k"):
        p = f"k{i}_"
        V, B = int(z[p + "V"]), int(z[p + "B"])
        d, s, w = graph(z, p)
        x = z[p + "x"]
        rp, col, val = R.to_csr(V, d, s, w)
        intra, inter, deg = R.decompose(V, d, s, w, B)
        for op in OPS:
            v, t = R.csr_aggregate(V, rp, col, val, x, op)
            assert same_float(v, z[p + f"csr_{op}"]), (i, op)
            assert np.array_equal(t, z[p + f"csr_{op}_touched"])
            vi, _ = R.csr_aggregate(V, *R.to_csr(V, *intra), x, op)
            assert same_float(vi, z[p + f"intra_{op}"]), (i, op)
            vc, _ = R.coo_aggregate(V, d, s, val, x, op)
            assert same_float(vc, z[p + f"coo_{op}"]), (i, op)
            assert same_float(R.aggregate_full(V, d, s, w, x, op), z[p + f"full_{op}"])
            if op != "max":
                ids, blocks, bt = R.to_blocks(V, *intra, B)
                vd, _ = R.dense_block_aggregate(V, B, ids, blocks, bt, x)
                assert same_float(vd, z[p + f"dense_{op}"]), (i, op)
            got = R.aggregate_decomposed_csr(V, intra, inter, deg, x, op)
            assert same_float(got, z[p + f"dec_{op}_csr_intra_blocked_csr_inter"]), (i, op)
        rd, rs, rw = R.canonical(V, s, d, w)
        bwd, _ = R.csr_aggregate(V, *R.to_csr(V, rd, rs, rw), x, "sum")
        assert same_float(bwd, z[p + "bwd"])


def test_c_restatement_of_reduction_order(kernels_golden):
    """csr_order.c (the order the CUDA kernel implements) == np.add.reduceat."""
    z = kernels_golden
    for i in z.cases("k"):
        p = f"k{i}_"
        V = int(z[p + "V"])
        d, s, w = graph(z, p)
        rp, col, _ = R.to_csr(V, d, s, w)
        got = obuild.csr_sum(rp, col, w, z[p + "x"])
        assert same_float(got, z[p + "csr_sum"]), i


def test_c_order_long_rows():
    rng = np.random.default_rng(5)
    for n in (1, 2, 7, 8, 9, 128, 129, 130, 255, 256, 257, 1000, 5001, 20000):
        F = 3
        x = rng.standard_normal((n, F)).astype(np.float32)
        val = rng.uniform(0.1, 2, n).astype(np.float32)
        rp = np.array([0, n], np.int32)
        col = np.arange(n, dtype=np.int32)
        got = obuild.csr_sum(rp, col, val, x)
        ref = np.add.reduceat(val[:, None] * x, [0], axis=0)
        assert same_float(got[0], ref[0]), n


def test_cluster_bfs_oracle(reorder_golden):
    z = reorder_golden
    for i in z.cases("r"):
        p = f"r{i}_"
        V, B = int(z[p + "V"]), int(z[p + "B"])
        if V > 400:
            continue  # the pure-Python restatement is for small graphs
        comm, perm = R.cluster_bfs(V, z[p + "dst"], z[p + "src"], B)
        assert np.array_equal(comm, z[p + "community"]), i
        assert np.array_equal(perm, z[p + "perm"]), i
        rd, rs, _ = R.apply_reorder(V, z[p + "dst"], z[p + "src"], z.get(p + "w"), perm)
        assert np.array_equal(rd, z[p + "re_dst"]) and np.array_equal(rs, z[p + "re_src"])


def test_partition_from_ids_oracle(reorder_golden):
    z = reorder_golden
    for i in range(4):
        comm, perm = R.partition_from_ids(z[f"lp{i}_ids"], int(z[f"lp{i}_B"]))
        assert np.array_equal(comm, z[f"lp{i}_community"])
        assert np.array_equal(perm, z[f"lp{i}_perm"])


def test_layer_goldens_vs_oracle(layers_golden):
    """The composed oracle's forward matches the reference layers (1e-5)."""
    from conftest import rel_error
    z = layers_golden
    for i in range(4):
        p = f"l{i}_"
        V = int(z[p + "V"])
        model = str(z[p + "model"])
        d, s, w = z[p + "dst"], z[p + "src"], z.get(p + "w")
        x, W = z[p + "x"], z[p + "weight"]
        agg = R.aggregate_full(V, d, s, w, x, "sum")
        if model == "gin":
            agg = np.float32(1.2) * x + agg
        assert rel_error(agg @ W, z[p + "out_full"]) < 1e-5


@pytest.mark.parametrize("skew", [1, 2])
def test_generator_oracle_exact_count(skew):
    (d, s), comm = osynth.community_graph(500, 4000, block_gen=16, p_intra=0.5, p_global=0.1,
                                          window=3, skew=skew, seed=3)
    assert d.size == 4000
    assert not np.any(d == s)
    keys = d.astype(np.int64) * 500 + s
    assert np.unique(keys).size == 4000
    assert comm.shape == (500,) and comm.max() == (500 + 15) // 16 - 1
    (d2, s2), _ = osynth.community_graph(500, 4000, block_gen=16, p_intra=0.5, p_global=0.1,
                                         window=3, skew=skew, seed=3)
    assert np.array_equal(d, d2) and np.array_equal(s, s2)
