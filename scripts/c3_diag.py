"""C3 training-step error anatomy (development): per pair, the loss and each
dW against the fp32 and fp64 oracle compositions."""
import pathlib
import sys

import numpy as np
import torch

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import bench  # noqa: E402
import paper_2305_17408_b200 as ag  # noqa: E402
from paper_2305_17408_b200 import synth as agsynth  # noqa: E402
from conftest import rel_error, to_np  # noqa: E402
import test_config_parity_gpu as T  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
rg, dec, net = T._workload(name)
V, dims = dec.num_vertices, net.dims
x = np.random.default_rng(0).standard_normal((V, dims[0])).astype(np.float32)
labels, mask = agsynth.labels_and_mask(V, dims[-1], seed=0)
ws = [to_np(w).copy() for w in net.weights]
oloss, og, oz = T._oracle_step(rg, net, x, ws, labels, mask)
eloss, eg, ez = T._oracle_step(rg, net, x, ws, labels, mask, np.float64)
print("logits |max|", float(np.abs(ez).max()), "oracle32 logits vs64", rel_error(oz, ez))
import bench as _b
print("oracle32 vs 64: loss", abs(oloss - eloss), "dW", [f"{rel_error(o, e):.2e}" for o, e in zip(og, eg)])
xt = torch.from_numpy(x).cuda()
lt = torch.from_numpy(labels.astype(np.int32)).cuda()
mt = torch.from_numpy(mask).cuda()
for pair in [None] + T.PAIRS:
    net.kernels.clear()
    if pair is None:
        net.autotune()
        label = "autotuned " + str({k: (a.value, b.value) for k, (a, b) in net.kernels.items()})
    else:
        net.default_pair = pair
        label = f"{pair[0].value}+{pair[1].value}"
    logits, _ = net.forward(xt)
    print(label, "logits vs32", rel_error(to_np(logits), oz), "vs64", rel_error(to_np(logits), ez))
    for eng in ("simt",):
        import paper_2305_17408_b200.models as M
        orig = M.gemm
        M.gemm = lambda *a, **k: orig(*a, **{**k, "engine": eng})
        lg2, _ = net.forward(xt)
        loss2, gr2 = net.train_step(xt, lt, mt, int(mask.sum()), lr=0.0)
        M.gemm = orig
        print("   simt-gemm logits vs64", rel_error(to_np(lg2), ez), "loss vs64", abs(float(loss2.item()) - eloss),
              "dW vs64", [f"{rel_error(to_np(g), e):.2e}" for g, e in zip(gr2, eg)])
    loss, grads = net.train_step(xt, lt, mt, int(mask.sum()), lr=0.0)
    print("   loss vs32", abs(float(loss.item()) - oloss), "vs64", abs(float(loss.item()) - eloss))
    print("   dW vs32", [f"{rel_error(to_np(g), o):.2e}" for g, o in zip(grads, og)],
          "vs64", [f"{rel_error(to_np(g), e):.2e}" for g, e in zip(grads, eg)], flush=True)
