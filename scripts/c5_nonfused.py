"""C5: the (dense_block, coo_atomic) pair unfused -- the coo role as the row
gather (ag_coo_gather_spmm) then the dense intra role combined into it --
against the fused slab launch (development)."""
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

cfg = bench.CONFIGS["C5"]
_, rg, dec, net, _ = bench.build_workload(cfg)
intra, inter = K.decomposed_execs(dec)
out = {}
for F in (256, 100, 48):
    x = torch.randn((rg.num_vertices, F), device="cuda")
    y = torch.empty_like(x)

    def unfused():
        inter.run_raw_into(ag.KernelKind.COO_ATOMIC, x, y, ag.AggregateOp.SUM, 0)
        intra.run_combine_into(ag.KernelKind.DENSE_BLOCK, x, y, ag.AggregateOp.SUM,
                               inter.csr.touched(), dec.full_in_degree, 0)

    r = {"unfused_gather": _time_ms(unfused, reps=5),
         "gather_only": _time_ms(lambda: inter.run_raw_into(ag.KernelKind.COO_ATOMIC, x, y,
                                                            ag.AggregateOp.SUM, 0), reps=5),
         "fused_slab": _time_ms(lambda: K.run_fused_pair(dec, x, y, ag.AggregateOp.SUM,
                                                          kernel_intra=ag.KernelKind.DENSE_BLOCK,
                                                          kernel_inter=ag.KernelKind.COO_ATOMIC),
                                reps=5)}
    out[F] = {k: round(v, 3) for k, v in r.items()}
    print(json.dumps(out), flush=True)
