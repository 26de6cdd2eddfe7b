"""GPU: bit-packed ReLU masks (include/adaptgear_b200.h "relu bits").

The training step stores each hidden activation's ReLU mask as one bit per
element, written by the epilogue that applies the ReLU (the update GEMM or the
slab aggregation) and read by the backward epilogues (the dH GEMM and the
transposed aggregation) instead of re-reading the fp32 activation.  Checked
here: the bit layout against numpy, every producer's bits against
ag_relu_bits of its own output, and every consumer against the fp32-mask
semantics (out = h > 0 ? out : 0), at widths that exercise partial words and
both slab lane layouts (VEC 1 / 2).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2305_17408_b200 as ag  # noqa: E402
from paper_2305_17408_b200 import kernels as K  # noqa: E402
from conftest import random_graph_arrays, rel_error, same_float, to_np  # noqa: E402
from oracle import ref_numpy as R  # noqa: E402

pytestmark = pytest.mark.gpu


def np_bits(h):
    rows, feat = h.shape
    w = (feat + 31) // 32
    pad = np.zeros((rows, w * 32), bool)
    pad[:, :feat] = h > 0
    b = pad.reshape(rows, w, 32).astype(np.uint64) << np.arange(32, dtype=np.uint64)
    return b.sum(axis=2).astype(np.uint32).view(np.int32)


@pytest.mark.parametrize("feat", [1, 31, 32, 33, 47, 100, 256])
def test_relu_bits_layout(rng, feat):
    h = rng.standard_normal((301, feat)).astype(np.float32)
    h[rng.random(h.shape) < 0.1] = 0.0  # exact zeros are "not > 0"
    got = to_np(K.relu_bits(torch.from_numpy(h).cuda()))
    assert np.array_equal(got, np_bits(h))


@pytest.mark.parametrize("N", [47, 48, 64, 256])
def test_gemm_mask_out_and_bit_mask(rng, N):
    M, Kd = 1000, 40
    a = torch.from_numpy(rng.standard_normal((M, Kd)).astype(np.float32)).cuda()
    w = torch.from_numpy(rng.standard_normal((Kd, N)).astype(np.float32)).cuda()
    base = torch.zeros((M, (N + 3) // 4 * 4), device="cuda")
    out = base[:, :N]
    bits = K.relu_bits_empty(M, N, "cuda")
    K.gemm(a, w, out, relu=True, mask_out=bits)
    assert torch.equal(bits, K.relu_bits(out))
    # consumer: dH = G W^T with the mask, as bits and as the fp32 activation
    g = torch.from_numpy(rng.standard_normal((M, 24)).astype(np.float32)).cuda()
    w2 = torch.from_numpy(rng.standard_normal((N, 24)).astype(np.float32)).cuda()
    d_bits = K.gemm(g, w2, trans_b=True, relu_mask_bits=bits)
    d_f32 = K.gemm(g, w2, trans_b=True, relu_mask=out.contiguous())
    ref = np.where(to_np(out) > 0, to_np(g) @ to_np(w2).T, 0)
    assert torch.equal(d_bits, d_f32)
    assert rel_error(to_np(d_bits), ref) < 1e-5
    for eng in ("simt",):  # the SIMT engine writes / reads the same layout
        bits2 = K.relu_bits_empty(M, N, "cuda")
        out2 = K.gemm(a, w, relu=True, engine=eng, mask_out=bits2)
        assert torch.equal(bits2, K.relu_bits(out2))
        d2 = K.gemm(g, w2, trans_b=True, relu_mask_bits=bits2, engine=eng)
        assert rel_error(to_np(d2), np.where(to_np(out2) > 0, to_np(g) @ to_np(w2).T, 0)) < 1e-5


@pytest.mark.parametrize("F", [33, 48, 64, 70, 100, 256])
def test_slab_relu_out_and_bit_mask(rng, F):
    V, d, s, _ = random_graph_arrays(rng, num_vertices=700, density=0.02)
    g = ag.gcn_normalize(ag.Graph.from_edges(V, d, s))
    dec = ag.decompose(ag.apply_reorder(g, ag.cluster_bfs(g, 16)), 16)
    x = torch.from_numpy(rng.standard_normal((V, F)).astype(np.float32)).cuda()
    h = torch.from_numpy(rng.standard_normal((V, F)).astype(np.float32)).cuda()
    hb = K.relu_bits(h)
    for ki, ke in [(ag.KernelKind.CSR_INTRA_BLOCKED, ag.KernelKind.CSR_INTER),
                   (ag.KernelKind.DENSE_BLOCK, ag.KernelKind.COO_ATOMIC)]:
        # producer: forward aggregation with the ReLU, bits of its output
        y = torch.empty_like(x)
        bits = K.relu_bits_empty(V, F, "cuda")
        K.run_fused_pair(dec, x, y, ag.AggregateOp.SUM, relu=True, kernel_intra=ki,
                         kernel_inter=ke, relu_out=bits)
        assert torch.equal(bits, K.relu_bits(y)), (F, ki)
        assert bool((y >= 0).all())
        # consumer: the bit mask equals the fp32 mask, bitwise
        y1, y2 = torch.empty_like(x), torch.empty_like(x)
        K.run_fused_pair(dec, x, y1, ag.AggregateOp.SUM, kernel_intra=ki, kernel_inter=ke,
                         relu_bits_in=hb)
        K.run_fused_pair(dec, x, y2, ag.AggregateOp.SUM, kernel_intra=ki, kernel_inter=ke,
                         relu_src=h)
        assert torch.equal(y1, y2)
        plain = torch.empty_like(x)
        K.run_fused_pair(dec, x, plain, ag.AggregateOp.SUM, kernel_intra=ki, kernel_inter=ke)
        assert torch.equal(y1, torch.where(h > 0, plain, torch.zeros_like(plain)))


def test_relu_bits_shape_checked():
    x = torch.zeros((10, 40), device="cuda")
    with pytest.raises(ValueError, match="relu bits"):
        K.gemm(x, torch.zeros((40, 40), device="cuda"), relu_mask_bits=torch.zeros(
            (10, 1), dtype=torch.int32, device="cuda"))
