"""The layers' update GEMM on the tensor cores (tcgen05 kind::tf32, 3xTF32)
against an fp64 reference of the same product, in the three operand layouts
the training step uses (forward agg @ W, dH = G W^T, dW = agg^T G), at ragged
sizes, with the fused ReLU / alpha / beta epilogue, and against the fp32 SIMT
kernel.  Tolerance: the reference's 1e-5 rel_error bar (conftest.py:22-26)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2305_17408_b200 import kernels as K  # noqa: E402
from conftest import rel_error, to_np  # noqa: E402

pytestmark = pytest.mark.gpu


def _ref(a, b, ta, tb):
    a64, b64 = a.double(), b.double()
    if ta:
        a64 = a64.t()
    if tb:
        b64 = b64.t()
    return a64 @ b64


# (M, K, N, trans_a, trans_b)
SHAPES = [
    (1000, 100, 256, False, False),   # layer-1 forward: agg[V,100] @ W[100,256]
    (777, 256, 256, False, False),    # hidden forward
    (513, 256, 48, False, False),     # last layer (padded class count)
    (300, 64, 32, False, False),
    (1000, 256, 256, False, True),    # dH = G @ W^T
    (257, 48, 256, False, True),      # dH of the last layer (K = padded classes)
    (256, 20000, 256, True, False),   # dW = agg^T @ G, split over K = V
    (100, 9000, 48, True, False),
    (64, 333, 16, True, False),
    (129, 31, 17, False, False),      # ragged everything
]


@pytest.mark.parametrize("M,Kd,N,ta,tb", SHAPES)
def test_tc_gemm_vs_fp64(M, Kd, N, ta, tb):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    a = torch.randn((Kd, M) if ta else (M, Kd), generator=g, device="cuda")
    b = torch.randn((N, Kd) if tb else (Kd, N), generator=g, device="cuda")
    if a.stride(0) % 4 or b.stride(0) % 4:
        pytest.skip("TMA needs 16-byte row strides")
    got = K.gemm(a, b, trans_a=ta, trans_b=tb, engine="tc")
    ref = _ref(a, b, ta, tb)
    # scale by sqrt(K): the products of N(0,1) operands grow like sqrt(K)
    err = rel_error(to_np(got) / np.sqrt(Kd), to_np(ref) / np.sqrt(Kd))
    assert err < 1e-5, err
    simt = K.gemm(a, b, trans_a=ta, trans_b=tb, engine="simt")
    assert rel_error(to_np(got) / np.sqrt(Kd), to_np(simt) / np.sqrt(Kd)) < 1e-5


def test_tc_gemm_epilogue_and_strides():
    g = torch.Generator(device="cuda").manual_seed(5)
    base = torch.randn((640, 136), generator=g, device="cuda")
    a = base[:, :128]                      # row stride 136 (not the width)
    w = torch.randn((128, 96), generator=g, device="cuda")
    c0 = torch.randn((640, 100), generator=g, device="cuda")
    full = c0.clone()
    out = full[:, :96]
    K.gemm(a, w, out, alpha=0.5, beta=2.0, relu=True, engine="tc")
    ref = torch.relu(0.5 * (a.double() @ w.double()) + 2.0 * c0[:, :96].double())
    assert rel_error(to_np(out), to_np(ref)) < 1e-5
    # the columns past the view are untouched
    assert torch.equal(full[:, 96:], c0[:, 96:])


def test_auto_engine_picks_simt_for_unaligned_strides():
    a = torch.randn((50, 47), device="cuda")   # 188-byte rows: no TMA
    w = torch.randn((47, 7), device="cuda")
    got = K.gemm(a, w)
    assert rel_error(to_np(got), to_np(a.double() @ w.double())) < 1e-5


@pytest.mark.parametrize("M,N,Kd,ta,tb", [(1000, 256, 256, False, False), (5000, 256, 48, False, True),
                                         (777, 200, 100, False, False), (256, 256, 70000, True, False)])
def test_tc_gemm_2sm_pairs_equal_single_sm(M, N, Kd, ta, tb, monkeypatch):
    """The opt-in 2-SM path (AG_TC_2SM=1: cta_group::2 MMAs, M = 256 over a CTA
    pair, each CTA holding half of the B tile) accumulates in the same order as
    the single-SM path: bitwise equal results, including partial tiles and
    the split-K dW shape."""
    g = torch.Generator(device="cuda").manual_seed(M + N)
    a = torch.randn((Kd, M) if ta else (M, Kd), device="cuda", generator=g)
    b = torch.randn((N, Kd) if tb else (Kd, N), device="cuda", generator=g)
    base = K.gemm(a, b, trans_a=ta, trans_b=tb, engine="tc")
    monkeypatch.setenv("AG_TC_2SM", "1")
    got = K.gemm(a, b, trans_a=ta, trans_b=tb, engine="tc")
    assert torch.equal(got, base)
