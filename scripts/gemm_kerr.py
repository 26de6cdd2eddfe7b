"""dW-shaped GEMM (out = A^T G, reduction over K rows) error against fp64 as K
grows, for the tensor-core 3xTF32 kernel and the fp32 SIMT kernel, next to
numpy's fp32 BLAS (the reference's arithmetic).  Development probe."""
import pathlib
import sys

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2305_17408_b200 import kernels as K  # noqa: E402

rng = np.random.default_rng(0)
for k in (1024, 16384, 169343, 1000000, 2449029):
    for m, n in ((64, 64), (256, 256)):
        a = rng.standard_normal((k, m)).astype(np.float32)
        g = (rng.standard_normal((k, n)) * 1e-3).astype(np.float32)
        ref = a.astype(np.float64).T @ g.astype(np.float64)
        scale = np.abs(a.astype(np.float64)).T @ np.abs(g.astype(np.float64))
        at, gt = torch.from_numpy(a).cuda(), torch.from_numpy(g).cuda()
        res = {}
        for eng in ("tc", "simt"):
            o = K.gemm(at, gt, trans_a=True, engine=eng).cpu().numpy().astype(np.float64)
            res[eng] = float((np.abs(o - ref) / scale).max())
        o = (a.T @ g).astype(np.float64)
        res["numpy"] = float((np.abs(o - ref) / scale).max())
        print(f"K={k} {m}x{n} err/sum|terms|: " + " ".join(f"{e}={v:.2e}" for e, v in res.items()),
              flush=True)

# device time of the C5 dW products (A = activations [V][M] M-major, G [V][N])
V = 2449029
for m, n in ((100, 256), (256, 256), (256, 48)):
    a = torch.randn((V, m), device="cuda")
    g = torch.randn((V, n), device="cuda")
    out = torch.empty((m, n), device="cuda")
    for _ in range(2):
        K.gemm(a, g, out, trans_a=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        K.gemm(a, g, out, trans_a=True)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"dW {m}x{n} K={V}: {ms:.3f} ms ({(m + n) * V * 4 / ms / 1e6:.0f} GB/s operand reads)",
          flush=True)
