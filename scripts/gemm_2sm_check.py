"""Development: the 2-SM (cta_group::2) GEMM path against the default path and
fp64, on the product shapes the training step uses."""
import os
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2305_17408_b200 import kernels as K  # noqa: E402


def rel(a, b):
    return float(((a.double() - b.double()).abs() / b.double().abs().clamp(min=1.0)).max())


torch.manual_seed(0)
for (M, N, Kd, ta, tb) in [(1000, 256, 256, False, False), (5000, 256, 48, False, True),
                           (4096, 256, 100, False, False), (777, 256, 256, False, True),
                           (256, 256, 70000, True, False), (100, 256, 70000, True, False)]:
    a = torch.randn((Kd, M) if ta else (M, Kd), device="cuda")
    b = torch.randn((N, Kd) if tb else (Kd, N), device="cuda")
    ref = (a.double().t() if ta else a.double()) @ (b.double().t() if tb else b.double())
    os.environ["AG_TC_2SM"] = "0"
    base = K.gemm(a, b, trans_a=ta, trans_b=tb)
    os.environ["AG_TC_2SM"] = "1"
    got = K.gemm(a, b, trans_a=ta, trans_b=tb)
    torch.cuda.synchronize()
    s = Kd ** 0.5
    print(f"M={M} N={N} K={Kd} ta={ta} tb={tb}: 2sm err {rel(got / s, ref / s):.2e} "
          f"base err {rel(base / s, ref / s):.2e}", flush=True)
