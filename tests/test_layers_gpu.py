"""GPU: the layer backward entry points (gcn_layer_backward / gin_layer_backward,
the north star's backward counterparts of models.py:86-112) and the loss
kernel's stride handling.

The backward formulas themselves are validated by central finite differences
on the CPU (tests/test_oracle_fd.py::test_layer_backward_formulas_...); here
the device entry points are compared with those formulas evaluated by the
oracle (numpy reduceat aggregation + fp32 matmuls) at 1e-5 rel, for a full
Graph subject and for a decomposed one with every kernel pair.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2305_17408_b200 as ag  # noqa: E402
from conftest import random_graph_arrays, rel_error, to_np  # noqa: E402
from oracle import ref_numpy as R  # noqa: E402

pytestmark = pytest.mark.gpu
K = ag.KernelKind
F32 = np.float32


def gemm_error(got, a, b):
    """max |got - a@b| / (|a| @ |b|): the GEMM's error relative to the sum of
    its terms' magnitudes (the standard fp32 dot-product bound; the fp64
    product is the reference).  fp32 accumulation gives ~K * 2^-24."""
    a64, b64 = np.asarray(a, np.float64), np.asarray(b, np.float64)
    ref = a64 @ b64
    scale = np.abs(a64) @ np.abs(b64)
    return float((np.abs(np.asarray(got, np.float64) - ref) / np.maximum(scale, 1e-30)).max())


def _setup(rng, model, V=300):
    V, d, s, _ = random_graph_arrays(rng, num_vertices=V, density=0.03)
    g = ag.Graph.from_edges(V, d, s)
    if model == "gcn":
        g = ag.gcn_normalize(g)
    rg = ag.apply_reorder(g, ag.cluster_bfs(g, 16))
    rt = rg.reverse()
    rd, rs = to_np(rg.dst), to_np(rg.src)
    rw = None if rg.weights is None else to_np(rg.weights)
    td, ts, tw = R.canonical(V, rs, rd, rw)
    return V, rg, rt, R.to_csr(V, td, ts, tw), R.to_csr(V, rd, rs, rw)


@pytest.mark.parametrize("subject", ["graph", "decomposed"])
def test_gcn_layer_backward_vs_oracle(rng, subject):
    V, rg, rt, bwd_csr, fwd_csr = _setup(rng, "gcn")
    params = ag.LayerParams.seeded("gcn", 24, 10, seed=4)
    x = rng.standard_normal((V, 24)).astype(F32)
    agg = R.csr_aggregate(V, *fwd_csr, x, "sum")[0]
    d_out = rng.standard_normal((V, 10)).astype(F32)
    w = np.asarray(params.weight, F32)
    ref_dw = (agg.T @ d_out).astype(F32)
    ref_dx = R.csr_aggregate(V, *bwd_csr, (d_out @ w.T).astype(F32), "sum")[0]
    subj = rt if subject == "graph" else ag.decompose(rt, 16)
    pairs = [(K.CSR_INTRA_BLOCKED, K.CSR_INTER)] if subject == "graph" else [
        (ki, ke) for ki in (K.CSR_INTRA_BLOCKED, K.DENSE_BLOCK) for ke in (K.CSR_INTER, K.COO_ATOMIC)]
    for ki, ke in pairs:
        d_x, d_w = ag.gcn_layer_backward(subj, x, agg, params, d_out, kernel_intra=ki,
                                         kernel_inter=ke)
        assert rel_error(to_np(d_w), ref_dw) < 1e-5, (ki, ke)
        assert rel_error(to_np(d_x), ref_dx) < 1e-5, (ki, ke)
    none_dx, d_w = ag.gcn_layer_backward(subj, x, agg, params, d_out, need_dx=False)
    assert none_dx is None and rel_error(to_np(d_w), ref_dw) < 1e-5


@pytest.mark.parametrize("subject", ["graph", "decomposed"])
def test_gin_layer_backward_vs_oracle(rng, subject):
    V, rg, rt, bwd_csr, fwd_csr = _setup(rng, "gin")
    params = ag.LayerParams.seeded("gin", 20, 12, seed=2, gin_eps=0.3)
    s = F32(params.gin_scale())
    x = rng.standard_normal((V, 20)).astype(F32)
    h = (s * x + R.csr_aggregate(V, *fwd_csr, x, "sum")[0]).astype(F32)
    d_out = rng.standard_normal((V, 12)).astype(F32)
    w = np.asarray(params.weight, F32)
    d_h = (d_out @ w.T).astype(F32)
    ref_dw = (h.T @ d_out).astype(F32)
    ref_dx = (s * d_h + R.csr_aggregate(V, *bwd_csr, d_h, "sum")[0]).astype(F32)
    subj = rt if subject == "graph" else ag.decompose(rt, 16)
    d_x, d_w = ag.gin_layer_backward(subj, x, h, params, d_out)
    # |h| reaches ~60 here (unweighted sums), so the K=300 reduction's fp32
    # rounding is measured against the sum of |terms| rather than |result|
    assert gemm_error(to_np(d_w), h.T, d_out) < 1e-6
    assert rel_error(to_np(d_x), ref_dx) < 1e-5
    # the forward it differentiates: ((1+eps) X + A X) W
    out = ag.gin_layer_forward(ag.decompose(rg, 16), x, params)
    assert gemm_error(to_np(out), h, w) < 1e-6


def test_layer_backward_rejects_wrong_model(rng):
    V, rg, rt, _, _ = _setup(rng, "gcn", V=64)
    x = np.zeros((V, 4), F32)
    with pytest.raises(ValueError):
        ag.gcn_layer_forward(rg, x, ag.LayerParams.seeded("gin", 4, 2))


@pytest.mark.parametrize("C", [7, 47, 100])
def test_softmax_xent_unpadded_logits(rng, C):
    """A contiguous [V, C] logits tensor (gemm() output, row stride C) with the
    padded [V, pad4(C)] gradient buffer GNN.loss_and_grad allocates: every
    gradient row lands at its own stride and the pad columns are 0."""
    V = 777
    logits = torch.from_numpy(rng.standard_normal((V, C)).astype(F32)).cuda()
    labels = rng.integers(0, C, V).astype(np.int32)
    mask = rng.random(V) < 0.5
    net = ag.GNN.__new__(ag.GNN)
    loss, d = ag.GNN.loss_and_grad(net, logits, torch.from_numpy(labels).cuda(),
                                   torch.from_numpy(mask).cuda(), int(mask.sum()))
    z = to_np(logits).astype(np.float64)
    z = z - z.max(axis=1, keepdims=True)
    p = np.exp(z) / np.exp(z).sum(axis=1, keepdims=True)
    rows = np.flatnonzero(mask)
    ref_loss = -np.log(p[rows, labels[rows]]).sum() / rows.size
    g = p.copy()
    g[rows, labels[rows]] -= 1.0
    g[~mask] = 0.0
    g /= rows.size
    assert abs(float(loss.item()) - ref_loss) <= 1e-5 * max(1.0, abs(ref_loss))
    assert rel_error(to_np(d), g) < 1e-6
    base = d.as_strided((V, d.stride(0)), (d.stride(0), 1))
    assert d.stride(0) == (C + 3) // 4 * 4
    assert not bool(base[:, C:].any())


def test_autotune_choice_cache_skips_profiling(rng, tmp_path):
    """GNN.autotune with a ChoiceCache: the first run profiles and stores the
    selector's locked pair and the pair that runs, keyed by graph hash, op,
    width and direction; a second network on the same topology reads both back
    without timing anything (selector.py:130-154 lock semantics, persisted)."""
    V, rg, rt, _, _ = _setup(rng, "gcn", V=400)
    dec = ag.decompose(rg, 16)
    net = ag.GNN.build("gcn", [24, 32, 5], dec, seed=1)
    cache = ag.ChoiceCache(tmp_path / "choices.json")
    first = net.autotune(cache=cache)
    assert cache.misses == len(first) and cache.hits == 0
    net2 = ag.GNN.build("gcn", [24, 32, 5], dec, seed=1, subject_t=net.subject_t)
    cache2 = ag.ChoiceCache(tmp_path / "choices.json")
    second = net2.autotune(cache=cache2)
    assert second == first and cache2.hits == len(first) and cache2.misses == 0
    assert net2.selector_choice == net.selector_choice
    # a different topology hashes to a different key
    assert ag.graph_key(dec) != ag.graph_key(net.subject_t)
