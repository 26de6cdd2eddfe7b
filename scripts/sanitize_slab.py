"""Small driver for compute-sanitizer (racecheck / synccheck / memcheck) over
every mode of the slab aggregation kernel (ag_fused.cu): the four fused
selector pairs (CSR x CSR = kModeSum3, dense_block x csr_inter = kModeDense3,
csr x coo = kModeSum3Coo, dense x coo = kModeDense3Coo), the generic and max
modes, with the GIN and ReLU-mask epilogues, at VEC 2 and VEC 1 widths.
Each launch is checked against the oracle so a race that corrupts values is
also caught.  Run under the sanitizer on the GPU box:

    compute-sanitizer --tool racecheck python scripts/sanitize_slab.py
"""
import pathlib
import sys

import numpy as np
import torch

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2305_17408_b200 as ag  # noqa: E402
from conftest import rel_error, same_float  # noqa: E402
from oracle import ref_numpy as R  # noqa: E402

K = ag.KernelKind
PAIRS = [(K.CSR_INTRA_BLOCKED, K.CSR_INTER), (K.DENSE_BLOCK, K.CSR_INTER),
         (K.CSR_INTRA_BLOCKED, K.COO_ATOMIC), (K.DENSE_BLOCK, K.COO_ATOMIC)]


def main(V=2500, E=30000, reps=1):
    rng = np.random.default_rng(3)
    keys = rng.choice(V * V, size=E, replace=False)
    g = ag.gcn_normalize(ag.Graph.from_edges(V, keys // V, keys % V))
    rg = ag.apply_reorder(g, ag.cluster_bfs(g, 16))
    dec = ag.decompose(rg, 16)
    intra = tuple(t.cpu().numpy() if t is not None else None
                  for t in (dec.intra.dst, dec.intra.src, dec.intra.weights))
    inter = tuple(t.cpu().numpy() if t is not None else None
                  for t in (dec.inter.dst, dec.inter.src, dec.inter.weights))
    deg = dec.full_in_degree.cpu().numpy()
    n = 0
    for F in (64, 256, 33):
        x = rng.standard_normal((V, F)).astype(np.float32)
        relu_src = rng.standard_normal((V, F)).astype(np.float32)
        xt, rt = torch.from_numpy(x).cuda(), torch.from_numpy(relu_src).cuda()
        ref = R.aggregate_decomposed_csr(V, intra, inter, deg, x, "sum")
        for _ in range(reps):
            for ki, ke in PAIRS:
                for gin, relu in ((None, None), (1.5, None), (None, rt)):
                    y = torch.empty_like(xt)
                    ag.kernels.run_fused_pair(dec, xt, y, ag.AggregateOp.SUM, gin, relu_src=relu,
                                      kernel_intra=ki, kernel_inter=ke)
                    want = ref if gin is None else np.float32(gin) * x + ref
                    if relu is not None:
                        want = np.where(relu_src > 0, want, 0).astype(np.float32)
                    got = y.cpu().numpy()
                    if (ki, ke) == PAIRS[0]:
                        assert same_float(got, want), (F, ki, ke, gin)
                    else:
                        assert rel_error(got, want) < 1e-5, (F, ki, ke, gin)
                    n += 1
            for op in (ag.AggregateOp.MEAN, ag.AggregateOp.MAX):
                got = ag.aggregate_decomposed(dec, xt, op, kernel_intra=K.CSR_INTRA_BLOCKED,
                                              kernel_inter=K.CSR_INTER).cpu().numpy()
                want = R.aggregate_decomposed_csr(V, intra, inter, deg, x, op.value)
                assert same_float(got, want), (F, op)
                n += 1
    torch.cuda.synchronize()
    print(f"sanitize_slab: {n} launches checked")


if __name__ == "__main__":
    main(reps=int(sys.argv[1]) if len(sys.argv) > 1 else 1)
