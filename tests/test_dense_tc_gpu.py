"""GPU: the tensor-core dense_block kernel (K4 on tcgen05, north star "a
tf32/bf16 mma variant with a stated tolerance").

The reference computes the intra role as a batched BLAS matmul over the
stored B x B diagonal blocks (kernels.py:228-250), order unpinned, pinned by
its tests at 1e-5 (test_kernels.py:139).  Here the blocks are packed into
block-diagonal 128-wide panels (8 blocks of 16, 4 of 32, 2 of 64, 1 of 128;
256-wide panels for B = 256) and multiplied on the tensor cores with 3xTF32
(ag_block_diag_gemm_tf32x3): stated tolerance 1e-5 rel against the oracle,
the reference's own bar for this kernel.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2305_17408_b200 as ag  # noqa: E402
from paper_2305_17408_b200 import kernels as K  # noqa: E402
from conftest import rel_error, to_np  # noqa: E402
from oracle import ref_numpy as R  # noqa: E402

pytestmark = pytest.mark.gpu


def _graph(B, V=1500, E=60000, seed=0, model="gcn"):
    from paper_2305_17408_b200 import synth
    g, comm = synth.community_graph(V, E, block_gen=B, p_intra=0.6, p_global=0.05, window=4,
                                    seed=seed)
    if model == "gcn":
        g = ag.gcn_normalize(g)
    rg = ag.apply_reorder(g, ag.reorder.partition_from_ids(comm, B))
    return rg, ag.decompose(rg, B)


@pytest.mark.parametrize("B", [16, 32, 64, 128, 256])
@pytest.mark.parametrize("F", [64, 100])
def test_dense_block_tc_vs_oracle(B, F):
    rg, dec = _graph(B)
    V = dec.num_vertices
    blk = ag.to_dense_blocks(dec.intra, B)
    x = np.random.default_rng(B + F).standard_normal((V, F)).astype(np.float32)
    ids, blocks, touched = (to_np(blk.community_ids), to_np(blk.blocks), to_np(blk.row_touched))
    ref, ref_t = R.dense_block_aggregate(V, B, ids, blocks, touched, x)
    got = K.aggregate_dense_block(blk, torch.from_numpy(x).cuda(), ag.AggregateOp.SUM,
                                  precision="tf32x3")
    assert rel_error(to_np(got.values), ref) < 1e-5
    assert np.array_equal(to_np(got.touched), ref_t)
    simt = K.aggregate_dense_block(blk, torch.from_numpy(x).cuda(), ag.AggregateOp.SUM,
                                   precision="fp32")
    assert rel_error(to_np(simt.values), ref) < 1e-5
    # the default picks the tensor cores from B = 64 up
    xt = torch.from_numpy(x).cuda()
    assert K.dense_block_engine(blk, xt, None) == ("tc" if B >= 64 else "simt")


@pytest.mark.parametrize("B", [64, 128, 256])
@pytest.mark.parametrize("op", [ag.AggregateOp.SUM, ag.AggregateOp.MEAN])
def test_decomposed_dense_block_tc_pair(B, op):
    """aggregate_decomposed(dense_block, csr_inter): the inter partial first,
    then the tensor-core block product accumulated onto it (combine(sum));
    mean keeps the SIMT kernel's fused divide.  1e-5 vs the dense oracle."""
    rg, dec = _graph(B, seed=1)
    V = dec.num_vertices
    x = np.random.default_rng(B).standard_normal((V, 64)).astype(np.float32)
    d, s = to_np(rg.dst), to_np(rg.src)
    w = None if rg.weights is None else to_np(rg.weights)
    ref = R.dense_reference(V, d, s, w, x, op.value)
    got = ag.aggregate_decomposed(dec, x, op, kernel_intra=ag.KernelKind.DENSE_BLOCK,
                                  kernel_inter=ag.KernelKind.CSR_INTER)
    assert rel_error(to_np(got), ref) < 1e-5


def test_dense_block_tc_rejects_bad_geometry():
    rg, dec = _graph(16, V=400, E=4000)
    blk = ag.to_dense_blocks(dec.intra, 16)
    xt = torch.zeros((400, 6), device="cuda")  # row stride 6: not TMA-addressable
    with pytest.raises(ag.KernelError):
        K.aggregate_dense_block(blk, xt, ag.AggregateOp.SUM, precision="tf32x3")
    with pytest.raises(ValueError):
        K.aggregate_dense_block(blk, xt, ag.AggregateOp.SUM, precision="bf16")
