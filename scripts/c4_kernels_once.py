"""One launch each of C4's (B = 512) dense_block tensor-core kernel and its coo
row gather at F = 128 (ncu target)."""
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2305_17408_b200 as ag  # noqa: E402
from paper_2305_17408_b200 import kernels as K  # noqa: E402

bench.COMM_SIZE = 512
cfg = bench.CONFIGS["C4"]
_, rg, dec, net, _ = bench.build_workload(cfg)
intra, inter = K.decomposed_execs(dec)
x = torch.randn((rg.num_vertices, 128), device="cuda")
y = torch.empty_like(x)
for _ in range(2):  # formats built on the first pass; ncu -c counts the second
    inter.run_raw_into(ag.KernelKind.COO_ATOMIC, x, y, ag.AggregateOp.SUM, 0)
    intra.run_combine_into(ag.KernelKind.DENSE_BLOCK, x, y, ag.AggregateOp.SUM,
                           inter.csr.touched(), dec.full_in_degree, 0)
torch.cuda.synchronize()
