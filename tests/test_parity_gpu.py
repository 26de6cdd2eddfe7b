"""GPU parity: the device path against the reference's golden vectors and the
oracle.  Bit-exact for every integer array and for the CSR kernels' floats
(they reproduce np.add.reduceat's order); tolerance-based (the reference's own
bars, test_kernels.py / test_acceptance.py) for COO (1e-4), dense blocks and
GEMMs (1e-5).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2305_17408_b200 as ag  # noqa: E402
from paper_2305_17408_b200 import kernels as K  # noqa: E402
from conftest import rel_error, same_float, to_np  # noqa: E402
from oracle import ref_numpy as R  # noqa: E402

pytestmark = pytest.mark.gpu
OPS = (ag.AggregateOp.SUM, ag.AggregateOp.MEAN, ag.AggregateOp.MAX)


def golden_graph(z, p, role=""):
    pre = p + (role + "_" if role else "")
    w = z.get(pre + "w")
    return ag.Graph.from_edges(int(z[p + "V"]), z[pre + "dst"], z[pre + "src"], w)


def test_canonicalize_and_formats_bit_exact(kernels_golden):
    z = kernels_golden
    for i in z.cases("k"):
        p = f"k{i}_"
        V = int(z[p + "V"])
        g = ag.Graph.from_edges(V, z[p + "raw_dst"], z[p + "raw_src"], z.get(p + "raw_w"))
        assert np.array_equal(to_np(g.dst), z[p + "dst"]), i
        assert np.array_equal(to_np(g.src), z[p + "src"]), i
        if z.get(p + "w") is not None:
            assert same_float(to_np(g.weights), z[p + "w"]), i
        a = ag.to_csr(g)
        assert np.array_equal(to_np(a.row_ptr), z[p + "row_ptr"])
        gn = ag.gcn_normalize(g)
        assert np.array_equal(to_np(gn.dst), z[p + "gcn_dst"])
        assert np.array_equal(to_np(gn.src), z[p + "gcn_src"])
        assert same_float(to_np(gn.weights), z[p + "gcn_w"]), i
        r = g.reverse()
        assert np.array_equal(to_np(r.dst), z[p + "rev_dst"])
        assert np.array_equal(to_np(r.src), z[p + "rev_src"])
        B = int(z[p + "B"])
        d = ag.decompose(g, B)
        for role, sub in (("intra", d.intra), ("inter", d.inter)):
            assert np.array_equal(to_np(sub.dst), z[p + role + "_dst"])
            assert np.array_equal(to_np(sub.src), z[p + role + "_src"])
            if z.get(p + role + "_w") is not None:
                assert same_float(to_np(sub.weights), z[p + role + "_w"])
        assert np.array_equal(to_np(d.full_in_degree), z[p + "full_in_degree"])
        blk = ag.to_dense_blocks(d.intra, B)
        assert np.array_equal(to_np(blk.community_ids), z[p + "blk_ids"])
        assert same_float(to_np(blk.blocks), z[p + "blk_blocks"])
        assert np.array_equal(to_np(blk.row_touched), z[p + "blk_touched"])


def test_csr_kernels_bitwise_vs_reference(kernels_golden):
    z = kernels_golden
    for i in z.cases("k"):
        p = f"k{i}_"
        g = golden_graph(z, p)
        B = int(z[p + "B"])
        x = z[p + "x"]
        a = ag.to_csr(g)
        d = ag.decompose(g, B)
        ia = ag.to_csr(d.intra)
        for op in OPS:
            o = op.value
            pr = ag.aggregate_csr_inter(a, x, op)
            assert same_float(to_np(pr.values), z[p + f"csr_{o}"]), (i, o)
            assert np.array_equal(to_np(pr.touched), z[p + f"csr_{o}_touched"])
            for budget in (1024, 48 * 1024, 1 << 40):
                pi = ag.aggregate_csr_intra_blocked(ia, x, op, B, tile_budget_bytes=budget)
                assert same_float(to_np(pi.values), z[p + f"intra_{o}"]), (i, o, budget)
            assert same_float(to_np(ag.aggregate_full(g, x, op)), z[p + f"full_{o}"]), (i, o)
            got = ag.aggregate_decomposed(d, x, op, kernel_intra=ag.KernelKind.CSR_INTRA_BLOCKED,
                                          kernel_inter=ag.KernelKind.CSR_INTER)
            assert same_float(to_np(got), z[p + f"dec_{o}_csr_intra_blocked_csr_inter"]), (i, o)
        bwd = ag.backward_sum(g.reverse(), x)
        assert same_float(to_np(bwd), z[p + "bwd"]), i


def test_coo_dense_and_pairs_within_tolerance(kernels_golden):
    z = kernels_golden
    for i in z.cases("k"):
        p = f"k{i}_"
        g = golden_graph(z, p)
        B = int(z[p + "B"])
        x = z[p + "x"]
        d = ag.decompose(g, B)
        for op in OPS:
            o = op.value
            c = ag.aggregate_coo_atomic(ag.to_coo(g), x, op)
            tol = 0.0 if op is ag.AggregateOp.MAX else 1e-4
            assert rel_error(to_np(c.values), z[p + f"coo_{o}"]) <= tol, (i, o)
            if op is ag.AggregateOp.MAX:
                assert c.note == "max via atomic compare-exchange emulation"
            else:
                db = ag.aggregate_dense_block(ag.to_dense_blocks(d.intra, B), x, op)
                assert rel_error(to_np(db.values), z[p + f"dense_{o}"]) < 1e-5, (i, o)
            for ki in (ag.KernelKind.CSR_INTRA_BLOCKED, ag.KernelKind.DENSE_BLOCK):
                if op is ag.AggregateOp.MAX and ki is ag.KernelKind.DENSE_BLOCK:
                    continue
                for ke in (ag.KernelKind.CSR_INTER, ag.KernelKind.COO_ATOMIC):
                    got = to_np(ag.aggregate_decomposed(d, x, op, kernel_intra=ki,
                                                        kernel_inter=ke))
                    ref = z[p + f"dec_{o}_{ki.value}_{ke.value}"]
                    tol = 0.0 if op is ag.AggregateOp.MAX else 1e-4
                    assert rel_error(got, ref) <= tol, (i, o, ki, ke)
            dref = z.get(p + f"dref_{o}")
            if dref is not None:
                got = to_np(ag.aggregate_dense_reference(g, x, op))
                assert rel_error(got, dref) <= (0.0 if op is ag.AggregateOp.MAX else 1e-5)


def test_kernel_errors():
    g = ag.Graph.from_edges(4, [3], [0])
    with pytest.raises(ag.KernelError, match="off-diagonal"):
        ag.aggregate_csr_intra_blocked(ag.to_csr(g), np.zeros((4, 1), np.float32),
                                       ag.AggregateOp.SUM, 2)
    with pytest.raises(ValueError, match="off-diagonal"):
        ag.to_dense_blocks(g, 2)
    g2 = ag.Graph.from_edges(2, [1], [0])
    with pytest.raises(ag.KernelError, match="max"):
        ag.aggregate_dense_block(ag.to_dense_blocks(g2, 2), np.ones((2, 1), np.float32),
                                 ag.AggregateOp.MAX)
    with pytest.raises(ag.KernelError):
        ag.aggregate_csr_inter(ag.to_csr(g), np.zeros((5, 2), np.float32), ag.AggregateOp.SUM)
    with pytest.raises(ag.KernelError, match="capped"):
        ag.aggregate_dense_reference(ag.Graph.from_edges(5000, [1], [0]),
                                     np.zeros((5000, 1), np.float32), ag.AggregateOp.SUM)
    with pytest.raises(ValueError, match="out of range"):
        ag.Graph.from_edges(3, [3], [0])
    a = ag.empty_partial(2, 1, ag.AggregateOp.SUM)
    b = ag.empty_partial(2, 1, ag.AggregateOp.MAX)
    with pytest.raises(ag.KernelError):
        ag.combine(a, b, ag.AggregateOp.SUM)
    with pytest.raises(ag.KernelError):
        m = ag.empty_partial(2, 1, ag.AggregateOp.MEAN)
        ag.combine(m, m, ag.AggregateOp.MEAN)
    ex = ag.SubgraphExec.for_inter(g, 4)
    with pytest.raises(ag.KernelError):
        ex.run(ag.KernelKind.DENSE_BLOCK, np.zeros((4, 2), np.float32), ag.AggregateOp.SUM)


def test_tiny_examples():
    g = ag.Graph.from_edges(3, [2, 2], [0, 1], [1.0, 2.0])
    x = np.array([[1.0], [10.0], [100.0]], dtype=np.float32)
    p = ag.aggregate_csr_inter(ag.to_csr(g), x, ag.AggregateOp.SUM)
    assert to_np(p.values).tolist() == [[0.0], [0.0], [21.0]]
    assert to_np(p.touched).tolist() == [False, False, True]
    intra = ag.empty_partial(4, 1, ag.AggregateOp.MAX)
    inter = ag.empty_partial(4, 1, ag.AggregateOp.MAX)
    intra.values[0], intra.touched[0] = -5.0, True
    inter.values[1], inter.touched[1] = -7.0, True
    intra.values[2], intra.touched[2] = -3.0, True
    inter.values[2], inter.touched[2] = -9.0, True
    out = ag.combine(intra, inter, ag.AggregateOp.MAX)
    assert to_np(out).tolist() == [[-5.0], [-7.0], [-3.0], [0.0]]
    e = ag.Graph.from_edges(3, [], [])
    c = ag.aggregate_coo_atomic(ag.to_coo(e), np.ones((3, 2), np.float32), ag.AggregateOp.SUM)
    assert not to_np(c.touched).any() and not to_np(c.values).any()
    assert to_np(ag.to_csr(e).row_ptr).tolist() == [0, 0, 0, 0]


def test_reorder_bit_exact(reorder_golden):
    z = reorder_golden
    for i in z.cases("r"):
        p = f"r{i}_"
        V, B = int(z[p + "V"]), int(z[p + "B"])
        g = ag.Graph.from_edges(V, z[p + "dst"], z[p + "src"], z.get(p + "w"))
        part = ag.cluster_bfs(g, B)
        assert np.array_equal(part.community_of, z[p + "community"]), i
        assert np.array_equal(part.permutation, z[p + "perm"]), i
        rg = ag.apply_reorder(g, part)
        assert np.array_equal(to_np(rg.dst), z[p + "re_dst"])
        assert np.array_equal(to_np(rg.src), z[p + "re_src"])
        if z.get(p + "re_w") is not None:
            assert same_float(to_np(rg.weights), z[p + "re_w"])


def test_layers_vs_reference(layers_golden):
    z = layers_golden
    for i in range(4):
        p = f"l{i}_"
        V, B = int(z[p + "V"]), int(z[p + "B"])
        model = str(z[p + "model"])
        g = ag.Graph.from_edges(V, z[p + "dst"], z[p + "src"], z.get(p + "w"))
        perm = z[p + "perm"]
        part = ag.Partition(V, np.zeros(V, np.int64), perm.astype(np.int64), B)
        d = ag.decompose(ag.apply_reorder(g, part), B)
        x = z[p + "x"]
        xp = np.empty_like(x)
        xp[perm] = x
        params = ag.LayerParams(model, x.shape[1], z[p + "weight"].shape[1],
                                z[p + "weight"].copy(), gin_eps=0.2)
        fwd = ag.gcn_layer_forward if model == "gcn" else ag.gin_layer_forward
        assert rel_error(to_np(fwd(d, xp, params)), z[p + "out_decomposed"]) < 1e-4
        assert rel_error(to_np(fwd(g, x, params)), z[p + "out_full"]) < 1e-5
    g = ag.Graph.from_edges(64, z["pipe_dst"], z["pipe_src"])
    x = z["pipe_x"]
    p_gcn = ag.LayerParams.seeded("gcn", 8, 8, seed=11)
    p_gin = ag.LayerParams.seeded("gin", 8, 8, seed=11, gin_eps=0.1)
    assert rel_error(to_np(ag.gcn_layer_forward(ag.gcn_normalize(g), x, p_gcn)),
                     z["pipe_gcn"]) < 1e-5
    assert rel_error(to_np(ag.gin_layer_forward(g, x, p_gin)), z["pipe_gin"]) < 1e-5


def test_random_graphs_vs_oracle(rng):
    """The reference's criterion-1 sweep shape, against the numpy oracle."""
    from conftest import random_graph_arrays
    for _ in range(40):
        weighted = bool(rng.integers(2))
        V, d, s, w = random_graph_arrays(rng, weighted=weighted)
        B = int(rng.integers(1, V + 1))
        F = int(rng.integers(1, 70))
        x = rng.standard_normal((V, F)).astype(np.float32)
        g = ag.Graph.from_edges(V, d, s, w)
        cd, cs, cw = R.canonical(V, d, s, w)
        dec = ag.decompose(g, B)
        for op in OPS:
            ref = R.aggregate_full(V, cd, cs, cw, x, op.value)
            assert same_float(to_np(ag.aggregate_full(g, x, op)), ref)
            if B <= 2048:
                got = ag.aggregate_decomposed(dec, x, op,
                                              kernel_intra=ag.KernelKind.CSR_INTRA_BLOCKED,
                                              kernel_inter=ag.KernelKind.CSR_INTER)
                intra, inter, deg = R.decompose(V, cd, cs, cw, B)
                assert same_float(to_np(got), R.aggregate_decomposed_csr(V, intra, inter, deg,
                                                                         x, op.value))


def test_high_degree_rows_bitwise():
    """Rows far beyond the 128-leaf: the pairwise recursion and a hub row."""
    rng = np.random.default_rng(9)
    V = 40000
    rows, cols = [], []
    for r, deg in ((0, 39999), (1, 5000), (2, 1024), (3, 129), (4, 57)):
        cols.append(rng.choice(V, size=deg, replace=False))
        rows.append(np.full(deg, r))
    d, s = np.concatenate(rows), np.concatenate(cols)
    for F, weighted in ((1, False), (64, True), (100, True), (602, False)):
        w = rng.uniform(0.1, 2.0, d.size).astype(np.float32) if weighted else None
        g = ag.Graph.from_edges(V, d, s, w)
        x = rng.standard_normal((V, F)).astype(np.float32)
        cd, cs, cw = R.canonical(V, d, s, w)
        ref, _ = R.csr_aggregate(V, *R.to_csr(V, cd, cs, cw), x, "sum")
        got = ag.aggregate_csr_inter(ag.to_csr(g), x, ag.AggregateOp.SUM).values
        assert same_float(to_np(got), ref), F


def test_generator_matches_oracle():
    from oracle import synth as osynth
    from paper_2305_17408_b200 import synth
    for skew in (1, 2):
        args = dict(block_gen=16, p_intra=0.5, p_global=0.1, window=3, skew=skew, seed=11)
        g, comm = synth.community_graph(700, 6000, **args)
        (d, s), comm_o = osynth.community_graph(700, 6000, **args)
        assert np.array_equal(to_np(g.dst), d) and np.array_equal(to_np(g.src), s)
        assert np.array_equal(comm, comm_o)


def test_selector_loop_on_device(rng):
    from conftest import random_graph_arrays
    V, d, s, w = random_graph_arrays(rng, num_vertices=300, density=0.05, weighted=True)
    g = ag.Graph.from_edges(V, d, s, w)
    dec = ag.decompose(g, 16)
    x = rng.standard_normal((V, 32)).astype(np.float32)
    res, st, trace = ag.run_training_loop(dec, x, ag.AggregateOp.SUM, 10)
    assert st.phase is ag.Phase.LOCKED and len(trace) == 10
    steady = [r for r in trace if not r.is_profiling]
    assert steady and all(r.kernel_intra is st.choice_intra for r in steady)
    cd, cs, cw = R.canonical(V, d, s, w)
    assert rel_error(to_np(res), R.dense_reference(V, cd, cs, cw, x, "sum")) < 1e-4
    with pytest.raises(ValueError, match="profiling budget"):
        ag.run_training_loop(dec, x, ag.AggregateOp.SUM, 3)


@pytest.mark.parametrize("model", ["gcn", "gin"])
def test_training_step_vs_composed_oracle(model, rng):
    """Teacher-forced step: loss and every dW vs the numpy composition (1e-5 rel)."""
    from conftest import random_graph_arrays
    V, d, s, _ = random_graph_arrays(rng, num_vertices=400, density=0.02)
    g = ag.Graph.from_edges(V, d, s)
    if model == "gcn":
        g = ag.gcn_normalize(g)
    part = ag.cluster_bfs(g, 16)
    rg = ag.apply_reorder(g, part)
    dec = ag.decompose(rg, 16)
    dims = [24, 32, 16, 5]
    net = ag.GNN.build(model, dims, dec, seed=3, gin_eps=0.1)
    x = rng.standard_normal((V, dims[0])).astype(np.float32)
    labels = rng.integers(0, dims[-1], V).astype(np.int32)
    mask = rng.random(V) < 0.5
    ws = [to_np(w).copy() for w in net.weights]
    xt = torch.from_numpy(x).cuda()
    loss, grads = net.train_step(xt, torch.from_numpy(labels).cuda(),
                                 torch.from_numpy(mask).cuda(), int(mask.sum()), lr=0.0)
    rd, rs, rw = to_np(rg.dst), to_np(rg.src), to_np(rg.weights) if rg.weights is not None else None
    fwd_csr = R.to_csr(V, rd, rs, rw)
    td, ts, tw = R.canonical(V, rs, rd, rw)
    bwd_csr = R.to_csr(V, td, ts, tw)
    adj_f = lambda h: R.csr_aggregate(V, *fwd_csr, h, "sum")[0]  # noqa: E731
    adj_b = lambda h: R.csr_aggregate(V, *bwd_csr, h, "sum")[0]  # noqa: E731
    oloss, ograds, _ = R.gnn_step(model, adj_f, adj_b, x, ws, labels, mask, gin_eps=0.1)
    assert abs(float(loss.item()) - oloss) <= 1e-5 * max(1.0, abs(oloss))
    for l, (gw, ow) in enumerate(zip(grads, ograds)):
        assert rel_error(to_np(gw), ow) < 1e-5, l


def test_prepare_matches_manual_pipeline(rng):
    """bench.prepare (bench.py:128-151): normalise, reorder, decompose + timings."""
    from conftest import random_graph_arrays
    V, d, s, _ = random_graph_arrays(rng, num_vertices=300, density=0.03)
    g = ag.Graph.from_edges(V, d, s)
    for reorder in ("bfs", "none"):
        cfg = ag.RunConfig(model="gcn", reorder=reorder, comm_size=8)
        run = ag.prepare(cfg, g)
        gn = ag.gcn_normalize(g)
        part = ag.cluster_bfs(gn, 8) if reorder == "bfs" else ag.identity_partition(V, 8)
        rg = ag.apply_reorder(gn, part)
        assert torch.equal(run.graph.dst, rg.dst) and torch.equal(run.graph.src, rg.src)
        assert run.decomposed.intra.num_edges == ag.decompose(rg, 8).intra.num_edges
        assert run.reorder_ms >= 0 and run.decompose_ms >= 0
    with pytest.raises(ValueError, match="unknown reorder"):
        ag.prepare(ag.RunConfig(reorder="metis"), g)


@pytest.mark.parametrize("pair", [("dense_block", "coo_atomic"), ("csr_intra_blocked", "coo_atomic"),
                                  ("dense_block", "csr_inter")])
@pytest.mark.parametrize("model", ["gcn", "gin"])
def test_training_step_fused_pairs_vs_composed_oracle(model, pair, rng):
    """The training step on each fused selector pair the autotune may lock (the
    C5 bench runs dense_block + coo_atomic at every width): loss and dW within
    1e-5 of the composed numpy oracle, as for the bitwise CSR pair."""
    from conftest import random_graph_arrays
    V, d, s, _ = random_graph_arrays(rng, num_vertices=500, density=0.03)
    g = ag.Graph.from_edges(V, d, s)
    if model == "gcn":
        g = ag.gcn_normalize(g)
    rg = ag.apply_reorder(g, ag.cluster_bfs(g, 16))
    dec = ag.decompose(rg, 16)
    dims = [24, 32, 16, 5]
    net = ag.GNN.build(model, dims, dec, seed=3, gin_eps=0.1)
    net.default_pair = tuple(ag.KernelKind(k) for k in pair)
    x = rng.standard_normal((V, dims[0])).astype(np.float32)
    labels = rng.integers(0, dims[-1], V).astype(np.int32)
    mask = rng.random(V) < 0.5
    ws = [to_np(w).copy() for w in net.weights]
    loss, grads = net.train_step(torch.from_numpy(x).cuda(), torch.from_numpy(labels).cuda(),
                                 torch.from_numpy(mask).cuda(), int(mask.sum()), lr=0.0)
    rd, rs, rw = to_np(rg.dst), to_np(rg.src), to_np(rg.weights) if rg.weights is not None else None
    fwd_csr = R.to_csr(V, rd, rs, rw)
    td, ts, tw = R.canonical(V, rs, rd, rw)
    bwd_csr = R.to_csr(V, td, ts, tw)
    adj_f = lambda h: R.csr_aggregate(V, *fwd_csr, h, "sum")[0]  # noqa: E731
    adj_b = lambda h: R.csr_aggregate(V, *bwd_csr, h, "sum")[0]  # noqa: E731
    oloss, ograds, _ = R.gnn_step(model, adj_f, adj_b, x, ws, labels, mask, gin_eps=0.1)
    assert abs(float(loss.item()) - oloss) <= 1e-5 * max(1.0, abs(oloss))
    for l, (gw, ow) in enumerate(zip(grads, ograds)):
        assert rel_error(to_np(gw), ow) < 1e-5, l


@pytest.mark.parametrize("model", ["gcn", "gin"])
def test_graphed_train_step_matches_eager(model, rng):
    """GraphedTrainStep (the step as one CUDA graph per input buffer) computes
    exactly the eager step: same loss and weights, bit for bit, after the same
    number of steps."""
    from conftest import random_graph_arrays
    V, d, s, _ = random_graph_arrays(rng, num_vertices=600, density=0.02)
    g = ag.Graph.from_edges(V, d, s)
    if model == "gcn":
        g = ag.gcn_normalize(g)
    dec = ag.decompose(ag.apply_reorder(g, ag.cluster_bfs(g, 16)), 16)
    dims = [24, 32, 16, 5]
    x = torch.from_numpy(rng.standard_normal((V, dims[0])).astype(np.float32)).cuda()
    labels = torch.from_numpy(rng.integers(0, dims[-1], V).astype(np.int32)).cuda()
    mask = torch.from_numpy(rng.random(V) < 0.5).cuda()
    n = int(mask.sum().item())
    eager = ag.GNN.build(model, dims, dec, seed=3)
    graphed_net = ag.GNN.build(model, dims, dec, seed=3)
    for _ in range(4):  # 1 warm-up + the upload replay + 2 replays below
        loss_e, _ = eager.train_step(x, labels, mask, n, lr=0.05)
    step = ag.GraphedTrainStep(graphed_net, [(x, labels, mask)], n, lr=0.05, warmup=1)
    step.step(0)
    loss_g = step.step(0)
    torch.cuda.synchronize()
    assert torch.equal(loss_g, loss_e)
    for we, wg in zip(eager.weights, graphed_net.weights):
        assert torch.equal(we, wg)


@pytest.mark.parametrize("F", [1, 6, 44, 128, 300])
@pytest.mark.parametrize("weighted", [True, False])
def test_coo_gather_matches_atomic_and_oracle(F, weighted, monkeypatch):
    """coo_atomic's sum partial as a row gather (ag_coo_gather_spmm): equal to
    the atomic kernel and the oracle within the reference's 1e-4, for every
    vector width / lane split (F = 1, 6, 44, 128, 300), rows without edges
    (written 0) and unweighted graphs."""
    from conftest import rel_error
    rng = np.random.default_rng(F)
    V = 2000
    d = rng.integers(0, V // 2, 30000)  # the upper half of the rows has no edges
    s = rng.integers(0, V, 30000)
    g = ag.Graph.from_edges(V, d, s)
    if weighted:
        g = ag.gcn_normalize(g)
    coo = K.to_coo(g)
    x = rng.standard_normal((V, F)).astype(np.float32)
    got = K.aggregate_coo_atomic(coo, x, ag.AggregateOp.SUM)
    monkeypatch.setenv("AG_COO_ATOMIC", "1")
    atomic = K.aggregate_coo_atomic(coo, x, ag.AggregateOp.SUM)
    dd, ss = to_np(g.dst), to_np(g.src)
    w = None if g.weights is None else to_np(g.weights)
    dense = R.dense_reference(V, dd, ss, w, x, "sum")
    assert rel_error(to_np(got.values), dense) < 1e-4
    assert rel_error(to_np(got.values), to_np(atomic.values)) < 1e-4
    assert torch.equal(got.touched, atomic.touched)
    if not weighted:  # (gcn_normalize adds self loops to every row)
        assert not to_np(got.values)[V // 2:].any()
