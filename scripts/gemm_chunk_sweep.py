"""dW GEMM chunked split-K sweep (development): time of the C5 dW products and
error vs fp64 at K = 2.45M for AG_TC_CHUNK_KB x AG_TC_CHUNK_BN."""
import os
import pathlib
import sys

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2305_17408_b200 import kernels as K  # noqa: E402

V = 2449029
rng = np.random.default_rng(0)
a_np = rng.standard_normal((V, 256)).astype(np.float32)
g_np = (rng.standard_normal((V, 256)) * 1e-3).astype(np.float32)
ref = a_np[:, :256].astype(np.float64).T @ g_np.astype(np.float64)
scale = np.abs(a_np.astype(np.float64)).T @ np.abs(g_np.astype(np.float64))
a = torch.from_numpy(a_np).cuda()
g = torch.from_numpy(g_np).cuda()
x100 = a[:, :100].contiguous()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


for kb in ("64", "128", "256", "512"):
    for bn in ("256", "128"):
        os.environ["AG_TC_CHUNK_KB"], os.environ["AG_TC_CHUNK_BN"] = kb, bn
        o = K.gemm(a, g, trans_a=True).cpu().numpy().astype(np.float64)
        err = float((np.abs(o - ref) / scale).max())
        t256 = t(lambda: K.gemm(a, g, trans_a=True))
        t100 = t(lambda: K.gemm(x100, g, trans_a=True))
        print(f"chunk_kb={kb} bn={bn}: 256x256 {t256:.3f} ms, 100x256 {t100:.3f} ms, err {err:.2e}",
              flush=True)
