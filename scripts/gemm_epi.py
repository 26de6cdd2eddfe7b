"""C5 update-GEMM timings (development): forward with / without the ReLU
bit-mask emission, dH with the bit mask vs the fp32 activation mask, dW."""
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2305_17408_b200 import kernels as K  # noqa: E402

V = 2449029


def t(fn, reps=7):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


h = torch.randn((V, 256), device="cuda")
x100 = torch.randn((V, 100), device="cuda")
w = torch.randn((256, 256), device="cuda")
w100 = torch.randn((100, 256), device="cuda")
w48 = torch.randn((256, 48), device="cuda")
q = torch.randn((V, 48), device="cuda")
g = torch.randn((V, 256), device="cuda")
out = torch.empty((V, 256), device="cuda")
bits = K.relu_bits_empty(V, 256, "cuda")
hb = K.relu_bits(h)
res = {
    "fwd_256x256_relu": t(lambda: K.gemm(h, w, out, relu=True)),
    "fwd_256x256_relu_maskout": t(lambda: K.gemm(h, w, out, relu=True, mask_out=bits)),
    "fwd_100x256_relu": t(lambda: K.gemm(x100, w100, out, relu=True)),
    "fwd_100x256_relu_maskout": t(lambda: K.gemm(x100, w100, out, relu=True, mask_out=bits)),
    "dH_48x256_bits": t(lambda: K.gemm(q, w48, out, trans_b=True, relu_mask_bits=hb)),
    "dH_48x256_nomask": t(lambda: K.gemm(q, w48, out, trans_b=True)),
    "dW_256x256": t(lambda: K.gemm(h, g, trans_a=True)),
    "dW_100x256": t(lambda: K.gemm(x100, g, trans_a=True)),
    "dW_256x48": t(lambda: K.gemm(h, q, trans_a=True)),
    "dH_256x256": t(lambda: K.gemm(g, w, out, trans_b=True, relu_mask_bits=hb)),
}
for k, v in res.items():
    print(f"{k}: {v:.3f} ms", flush=True)
