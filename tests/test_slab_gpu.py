"""The slab aggregation kernel (ag_fused_spmm) on graphs that exercise each of
its source paths -- X ring, staged far ring, far-ring overflow to global
memory, rows past the 64-pair window, partial column tiles, the cp.async
(non-TMA) producers, several row ranges per CTA -- bitwise against the numpy
restatement of the reference's CSR kernels + combine (kernels.py:87-189,
:253-276), for every op.  The ring geometry (`window`) must never change a
value: the same aggregation with the window forced to 0 (every inter source
far) is bitwise identical."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2305_17408_b200 as ag  # noqa: E402
from paper_2305_17408_b200 import kernels as K  # noqa: E402
from paper_2305_17408_b200.decompose import full_graph  # noqa: E402
from oracle import ref_numpy as R  # noqa: E402
from conftest import same_float, to_np  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _slab_only(monkeypatch):
    """These graphs are small enough for the gather pair (ag_gather_pair_spmm,
    tests/test_gather_gpu.py); here the slab kernel's own modes are tested."""
    monkeypatch.setenv("AG_GATHER", "0")
OPS = (ag.AggregateOp.SUM, ag.AggregateOp.MEAN, ag.AggregateOp.MAX)


def _community(V, E, window, p_global, model="gcn", B=16, seed=0):
    from paper_2305_17408_b200 import synth
    g, comm = synth.community_graph(V, E, block_gen=B, p_intra=0.4, p_global=p_global,
                                    window=window, seed=seed)
    if model == "gcn":
        g = ag.gcn_normalize(g)
    rg = ag.apply_reorder(g, ag.reorder.partition_from_ids(comm, B))
    return rg, ag.decompose(rg, B)


def _oracle_pair(rg, B, x, op):
    V = rg.num_vertices
    d, s = to_np(rg.dst), to_np(rg.src)
    w = None if rg.weights is None else to_np(rg.weights)
    intra, inter, deg = R.decompose(V, d, s, w, B)
    return R.aggregate_decomposed_csr(V, intra, inter, deg, x, op)


def _pair(dec, x, op):
    return to_np(ag.aggregate_decomposed(dec, x, op, kernel_intra=ag.KernelKind.CSR_INTRA_BLOCKED,
                                         kernel_inter=ag.KernelKind.CSR_INTER))


def _force_window(dec, window):
    """Rebuild the cached slab layout of the decomposed graph's full CSR."""
    csr = K.to_csr(full_graph(dec))
    csr._window = window
    csr._codes = {}


@pytest.mark.parametrize("F", [7, 64, 100, 256])
def test_locality_graph_every_op_bitwise(F):
    rg, dec = _community(6000, 90000, window=6, p_global=0.05)
    x = np.random.default_rng(F).standard_normal((rg.num_vertices, F)).astype(np.float32)
    assert K.to_csr(full_graph(dec)).window() >= 6
    for op in OPS:
        assert same_float(_pair(dec, x, op), _oracle_pair(rg, 16, x, op.value)), (F, op)


def test_window_never_changes_values():
    rg, dec = _community(5000, 80000, window=8, p_global=0.05, model="gin")
    x = np.random.default_rng(1).standard_normal((rg.num_vertices, 64)).astype(np.float32)
    want = _pair(dec, x, ag.AggregateOp.SUM)
    for window in (0, 2, 16):
        _force_window(dec, window)
        got = _pair(dec, x, ag.AggregateOp.SUM)
        assert same_float(got, want), window
    assert same_float(want, _oracle_pair(rg, 16, x, "sum"))


def test_far_ring_overflow_and_long_rows():
    """No locality (every inter source far, far more than the far ring holds per
    block) plus hub rows far past the 64-pair window and the 128-item leaf."""
    rng = np.random.default_rng(3)
    V = 3000
    keys = rng.choice(V * V, size=60000, replace=False)
    d, s = keys // V, keys % V
    hub = rng.choice(V, size=900, replace=False)
    d = np.concatenate([d, np.full(hub.size, 5)])
    s = np.concatenate([s, hub])
    g = ag.gcn_normalize(ag.Graph.from_edges(V, d, s))
    dec = ag.decompose(g, 16)
    for F in (32, 100):
        x = rng.standard_normal((V, F)).astype(np.float32)
        for op in OPS:
            assert same_float(_pair(dec, x, op), _oracle_pair(g, 16, x, op.value)), (F, op)


def test_many_ranges_and_no_tma_path(monkeypatch):
    rg, dec = _community(40000, 400000, window=10, p_global=0.03)
    x = np.random.default_rng(5).standard_normal((rg.num_vertices, 96)).astype(np.float32)
    want = _oracle_pair(rg, 16, x, "sum")
    assert same_float(_pair(dec, x, ag.AggregateOp.SUM), want)
    monkeypatch.setenv("AG_SLAB_NO_TMA", "1")
    assert same_float(_pair(dec, x, ag.AggregateOp.SUM), want)
    monkeypatch.setenv("AG_SLAB_VEC", "1")
    assert same_float(_pair(dec, x, ag.AggregateOp.SUM), want)


def test_gin_and_relu_epilogues_bitwise():
    rg, dec = _community(4000, 50000, window=5, p_global=0.05, model="gin")
    rng = np.random.default_rng(8)
    x = torch.from_numpy(rng.standard_normal((rg.num_vertices, 64)).astype(np.float32)).cuda()
    h = torch.from_numpy(rng.standard_normal((rg.num_vertices, 64)).astype(np.float32)).cuda()
    y = torch.empty_like(x)
    K.run_fused_pair(dec, x, y, ag.AggregateOp.SUM, 1.25, relu_src=h)
    agg = _oracle_pair(rg, 16, to_np(x), "sum")
    want = np.float32(1.25) * to_np(x) + agg
    want = np.where(to_np(h) > 0, want, np.float32(0.0))
    assert same_float(to_np(y), want)


def test_gemm_raw_hi_is_bitwise_masked_split(monkeypatch):
    """kind::tf32 reads only the top 19 bits of an fp32 operand, so leaving x
    in place as the 'hi' half equals masking it (AG_TC_RAWHI)."""
    rng = np.random.default_rng(2)
    a = torch.from_numpy(rng.standard_normal((777, 256)).astype(np.float32)).cuda()
    b = torch.from_numpy(rng.standard_normal((256, 256)).astype(np.float32)).cuda()
    monkeypatch.setenv("AG_TC_RAWHI", "0")
    want = K.gemm(a, b)
    monkeypatch.setenv("AG_TC_RAWHI", "1")
    assert torch.equal(K.gemm(a, b), want)
    # a dW-shaped product (both operands split in shared memory, split K)
    h = torch.from_numpy(rng.standard_normal((300000, 64)).astype(np.float32)).cuda()
    g = torch.from_numpy(rng.standard_normal((300000, 48)).astype(np.float32)).cuda()
    assert g.numel() > K.PRESPLIT_MAX_ELEMS
    monkeypatch.setenv("AG_TC_RAWHI", "0")
    want = K.gemm(h, g, trans_a=True)
    monkeypatch.setenv("AG_TC_RAWHI", "1")
    assert torch.equal(K.gemm(h, g, trans_a=True), want)


@pytest.mark.parametrize("F", [64, 100, 256])
def test_dense_intra_pair_within_tolerance(F):
    """(dense_block, csr_inter) in one slab launch: the intra role as a dense
    16 x 16 block product (order-unpinned like the reference's BLAS matmul,
    kernels.py:247), the inter role bitwise -- against the reference pair."""
    from conftest import rel_error
    rg, dec = _community(6000, 90000, window=6, p_global=0.05)
    x = np.random.default_rng(F).standard_normal((rg.num_vertices, F)).astype(np.float32)
    got = to_np(ag.aggregate_decomposed(dec, x, ag.AggregateOp.SUM,
                                        kernel_intra=ag.KernelKind.DENSE_BLOCK,
                                        kernel_inter=ag.KernelKind.CSR_INTER))
    assert rel_error(got, _oracle_pair(rg, 16, x, "sum")) < 1e-5


@pytest.mark.parametrize("F", [48, 100, 256])
def test_dense_intra_large_graph(F):
    """Enough blocks per CTA that the two dense warps drift apart (each has its
    own weight staging buffer); against the bitwise CSR pair."""
    from conftest import rel_error
    rg, dec = _community(300000, 4000000, window=12, p_global=0.05)
    x = torch.randn((rg.num_vertices, F), device="cuda")
    want = torch.empty_like(x)
    K.run_fused_pair(dec, x, want, ag.AggregateOp.SUM)
    for ke in (ag.KernelKind.CSR_INTER, ag.KernelKind.COO_ATOMIC):
        y = torch.empty_like(x)
        for _ in range(3):
            K.run_fused_pair(dec, x, y, ag.AggregateOp.SUM, kernel_intra=ag.KernelKind.DENSE_BLOCK,
                             kernel_inter=ke)
            assert rel_error(to_np(y), to_np(want)) < 1e-5, ke


def test_dense_intra_epilogues():
    from conftest import rel_error
    rg, dec = _community(4000, 50000, window=5, p_global=0.05, model="gin")
    rng = np.random.default_rng(4)
    x = torch.from_numpy(rng.standard_normal((rg.num_vertices, 64)).astype(np.float32)).cuda()
    h = torch.from_numpy(rng.standard_normal((rg.num_vertices, 64)).astype(np.float32)).cuda()
    y = torch.empty_like(x)
    K.run_fused_pair(dec, x, y, ag.AggregateOp.SUM, 1.25, relu_src=h, dense_intra=True)
    want = np.float32(1.25) * to_np(x) + _oracle_pair(rg, 16, to_np(x), "sum")
    want = np.where(to_np(h) > 0, want, np.float32(0.0))
    assert rel_error(to_np(y), want) < 1e-5


COO_PAIRS = [(ag.KernelKind.CSR_INTRA_BLOCKED, ag.KernelKind.COO_ATOMIC),
             (ag.KernelKind.DENSE_BLOCK, ag.KernelKind.COO_ATOMIC)]


@pytest.mark.parametrize("F", [7, 64, 100, 256])
@pytest.mark.parametrize("pair", COO_PAIRS, ids=lambda p: p[0].value)
def test_coo_inter_pair_within_tolerance(F, pair):
    """(intra, coo_atomic) in one slab launch: the inter role in any order
    (AG_EPI_INTER_COO, like the reference's scrambled bincount) -- within the
    reference's 1e-4 (checked at 1e-5) of the bitwise pair."""
    from conftest import rel_error
    rg, dec = _community(6000, 90000, window=6, p_global=0.05)
    x = np.random.default_rng(F).standard_normal((rg.num_vertices, F)).astype(np.float32)
    got = to_np(ag.aggregate_decomposed(dec, x, ag.AggregateOp.SUM, kernel_intra=pair[0],
                                        kernel_inter=pair[1]))
    assert rel_error(got, _oracle_pair(rg, 16, x, "sum")) < 1e-5


@pytest.mark.parametrize("pair", COO_PAIRS, ids=lambda p: p[0].value)
def test_coo_inter_general_path_and_unweighted(pair):
    """Far-ring overflow, hub rows past the window (general path) and an
    unweighted (GIN) graph."""
    from conftest import rel_error
    rng = np.random.default_rng(3)
    V = 3000
    keys = rng.choice(V * V, size=60000, replace=False)
    d, s = keys // V, keys % V
    hub = rng.choice(V, size=900, replace=False)
    d = np.concatenate([d, np.full(hub.size, 5)])
    s = np.concatenate([s, hub])
    for g in (ag.gcn_normalize(ag.Graph.from_edges(V, d, s)), ag.Graph.from_edges(V, d, s)):
        dec = ag.decompose(g, 16)
        for F in (32, 100):
            x = rng.standard_normal((V, F)).astype(np.float32)
            got = to_np(ag.aggregate_decomposed(dec, x, ag.AggregateOp.SUM,
                                                kernel_intra=pair[0], kernel_inter=pair[1]))
            # a 900-edge hub row summed in fp32: the reference's coo bar (1e-4)
            assert rel_error(got, _oracle_pair(g, 16, x, "sum")) < 1e-4, F


@pytest.mark.parametrize("pair", COO_PAIRS, ids=lambda p: p[0].value)
def test_coo_inter_epilogues(pair):
    from conftest import rel_error
    rg, dec = _community(4000, 50000, window=5, p_global=0.05, model="gin")
    rng = np.random.default_rng(4)
    x = torch.from_numpy(rng.standard_normal((rg.num_vertices, 64)).astype(np.float32)).cuda()
    h = torch.from_numpy(rng.standard_normal((rg.num_vertices, 64)).astype(np.float32)).cuda()
    y = torch.empty_like(x)
    K.run_fused_pair(dec, x, y, ag.AggregateOp.SUM, 1.25, relu_src=h, kernel_intra=pair[0],
                     kernel_inter=pair[1])
    want = np.float32(1.25) * to_np(x) + _oracle_pair(rg, 16, to_np(x), "sum")
    want = np.where(to_np(h) > 0, want, np.float32(0.0))
    assert rel_error(to_np(y), want) < 1e-5


def test_coo_inter_needs_sum():
    rg, dec = _community(2000, 20000, window=4, p_global=0.05)
    x = torch.randn((rg.num_vertices, 16), device="cuda")
    y = torch.empty_like(x)
    with pytest.raises(ag.KernelError, match="no fused kernel"):
        K.run_fused_pair(dec, x, y, ag.AggregateOp.MEAN, kernel_inter=ag.KernelKind.COO_ATOMIC)
    # the unfused pair still serves mean / max
    for op in (ag.AggregateOp.MEAN, ag.AggregateOp.MAX):
        got = to_np(ag.aggregate_decomposed(dec, x, op,
                                            kernel_inter=ag.KernelKind.COO_ATOMIC))
        from conftest import rel_error
        assert rel_error(got, _oracle_pair(rg, 16, to_np(x), op.value)) < 1e-4
