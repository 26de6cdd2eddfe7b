"""One C5-shaped update GEMM (development: ncu / trace target).
    python scripts/gemm_one.py dh48 | fwd256 | fwd100 | dw256"""
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2305_17408_b200 import kernels as K  # noqa: E402

V = 2449029
which = sys.argv[1]
out = torch.empty((V, 256), device="cuda")
if which == "dh48":
    q = torch.randn((V, 48), device="cuda")
    w48 = torch.randn((256, 48), device="cuda")
    hb = K.relu_bits(torch.randn((V, 256), device="cuda"))
    fn = lambda: K.gemm(q, w48, out, trans_b=True, relu_mask_bits=hb)  # noqa: E731
elif which == "fwd256":
    h = torch.randn((V, 256), device="cuda")
    w = torch.randn((256, 256), device="cuda")
    bits = K.relu_bits_empty(V, 256, "cuda")
    fn = lambda: K.gemm(h, w, out, relu=True, mask_out=bits)  # noqa: E731
elif which == "fwd100":
    x = torch.randn((V, 100), device="cuda")
    w = torch.randn((100, 256), device="cuda")
    bits = K.relu_bits_empty(V, 256, "cuda")
    fn = lambda: K.gemm(x, w, out, relu=True, mask_out=bits)  # noqa: E731
else:
    h = torch.randn((V, 256), device="cuda")
    g = torch.randn((V, 256), device="cuda")
    fn = lambda: K.gemm(h, g, trans_a=True)  # noqa: E731
fn()
torch.cuda.synchronize()
