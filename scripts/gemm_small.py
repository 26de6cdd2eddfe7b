"""Development: the C5 skinny products (V x 256 x 48 forward, dW 256 x 48, masked dH
48 -> 256, V x 100 x 256) under the GEMM's environment knobs."""
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2305_17408_b200 import kernels as K  # noqa: E402
from paper_2305_17408_b200.models import _time_ms  # noqa: E402

V = 2449029
h = torch.randn((V, 256), device="cuda")
x100 = torch.randn((V, 100), device="cuda")
w48 = torch.randn((256, 48), device="cuda")
w100 = torch.randn((100, 256), device="cuda")
q = torch.randn((V, 48), device="cuda")
out48 = torch.empty((V, 48), device="cuda")
out = torch.empty((V, 256), device="cuda")
hb = K.relu_bits(h)
bits = K.relu_bits_empty(V, 256, "cuda")
r = {"fwd_256x48": _time_ms(lambda: K.gemm(h, w48, out48), reps=7),
     "dW_256x48": _time_ms(lambda: K.gemm(h, q, trans_a=True), reps=7),
     "dH_48x256": _time_ms(lambda: K.gemm(q, w48, out, trans_b=True, relu_mask_bits=hb), reps=7),
     "fwd_100x256": _time_ms(lambda: K.gemm(x100, w100, out, relu=True, mask_out=bits), reps=7)}
print({k: round(v, 3) for k, v in r.items()}, flush=True)
