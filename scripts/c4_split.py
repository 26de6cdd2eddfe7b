"""C4 (B = 512) aggregation split: the dense_block (tensor-core) intra role,
the coo_atomic inter role, and the combine, each timed alone (development)."""
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2305_17408_b200 as ag  # noqa: E402
from paper_2305_17408_b200 import kernels as K  # noqa: E402
from paper_2305_17408_b200.models import _time_ms  # noqa: E402

bench.COMM_SIZE = int(sys.argv[1]) if len(sys.argv) > 1 else 512
cfg = bench.CONFIGS["C4"]
_, rg, dec, net, _ = bench.build_workload(cfg)
intra_x, inter_x = K.decomposed_execs(dec)
out = {"B": bench.COMM_SIZE, "intra_edges": dec.intra.num_edges, "inter_edges": dec.inter.num_edges}
for F in (128, 44):
    x = torch.randn((rg.num_vertices, F), device="cuda")
    r = {}
    r["dense_block"] = _time_ms(lambda: intra_x.run(ag.KernelKind.DENSE_BLOCK, x, ag.AggregateOp.SUM), reps=5)
    r["csr_intra_blocked"] = _time_ms(lambda: intra_x.run(ag.KernelKind.CSR_INTRA_BLOCKED, x, ag.AggregateOp.SUM), reps=3)
    r["coo_atomic"] = _time_ms(lambda: inter_x.run(ag.KernelKind.COO_ATOMIC, x, ag.AggregateOp.SUM), reps=5)
    r["csr_inter"] = _time_ms(lambda: inter_x.run(ag.KernelKind.CSR_INTER, x, ag.AggregateOp.SUM), reps=3)
    r["pair_dense_coo"] = _time_ms(lambda: ag.aggregate_decomposed(dec, x, ag.AggregateOp.SUM, kernel_intra=ag.KernelKind.DENSE_BLOCK, kernel_inter=ag.KernelKind.COO_ATOMIC), reps=5)
    out[F] = {k: round(v, 3) for k, v in r.items()}
    print(json.dumps(out), flush=True)
