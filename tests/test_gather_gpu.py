"""The (dense_block, coo_atomic) selector pair on small graphs as one
order-free row gather over the full CSR (ag_gather_pair_spmm): against the
numpy restatement of the reference pair (kernels.py:228-250 dense intra,
:192-225 coo inter, :253-276 combine) at 1e-5 and against the slab kernel's
dense + coo mode, for every lane split and every epilogue (GIN (1+eps) x,
ReLU with its bit mask, the ReLU-backward mask)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2305_17408_b200 as ag  # noqa: E402
from paper_2305_17408_b200 import kernels as K  # noqa: E402
from oracle import ref_numpy as R  # noqa: E402
from conftest import rel_error, to_np  # noqa: E402

pytestmark = pytest.mark.gpu
DENSE_COO = dict(kernel_intra=ag.KernelKind.DENSE_BLOCK, kernel_inter=ag.KernelKind.COO_ATOMIC)


def _community(V, E, model="gcn", seed=0):
    from paper_2305_17408_b200 import synth
    g, comm = synth.community_graph(V, E, block_gen=16, p_intra=0.4, p_global=0.05, window=6,
                                    seed=seed)
    if model == "gcn":
        g = ag.gcn_normalize(g)
    rg = ag.apply_reorder(g, ag.reorder.partition_from_ids(comm, 16))
    return rg, ag.decompose(rg, 16)


def _oracle_pair(rg, x):
    V = rg.num_vertices
    d, s = to_np(rg.dst), to_np(rg.src)
    w = None if rg.weights is None else to_np(rg.weights)
    intra, inter, deg = R.decompose(V, d, s, w, 16)
    return R.aggregate_decomposed_csr(V, intra, inter, deg, x, "sum")


@pytest.mark.parametrize("F", [4, 16, 44, 64, 100, 256])
def test_gather_pair_matches_oracle_and_slab(F, monkeypatch):
    rg, dec = _community(5003, 70000)
    x = np.random.default_rng(F).standard_normal((rg.num_vertices, F)).astype(np.float32)
    got = to_np(ag.aggregate_decomposed(dec, x, ag.AggregateOp.SUM, **DENSE_COO))
    assert rel_error(got, _oracle_pair(rg, x)) < 1e-5
    monkeypatch.setenv("AG_GATHER", "0")
    slab = to_np(ag.aggregate_decomposed(dec, x, ag.AggregateOp.SUM, **DENSE_COO))
    assert rel_error(got, slab) < 1e-5


@pytest.mark.parametrize("F", [16, 48, 100])
def test_gather_pair_epilogues(F):
    rg, dec = _community(4001, 50000, model="gin", seed=3)
    rng = np.random.default_rng(4)
    V = rg.num_vertices
    x = torch.from_numpy(rng.standard_normal((V, F)).astype(np.float32)).cuda()
    h = torch.from_numpy(rng.standard_normal((V, F)).astype(np.float32)).cuda()
    y = torch.empty_like(x)
    K.run_fused_pair(dec, x, y, ag.AggregateOp.SUM, 1.25, relu_src=h, **DENSE_COO)
    want = np.float32(1.25) * to_np(x) + _oracle_pair(rg, to_np(x))
    want = np.where(to_np(h) > 0, want, np.float32(0.0))
    assert rel_error(to_np(y), want) < 1e-5
    bits = K.relu_bits_empty(V, F, x.device)
    y2 = torch.empty_like(x)
    K.run_fused_pair(dec, x, y2, ag.AggregateOp.SUM, relu=True, relu_out=bits, **DENSE_COO)
    assert rel_error(to_np(y2), np.maximum(_oracle_pair(rg, to_np(x)), 0)) < 1e-5
    assert torch.equal(bits, K.relu_bits(y2))
