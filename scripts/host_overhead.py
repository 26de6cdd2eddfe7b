"""Development: host (launch-side) time of one eager training step, GNN and the
row-partitioned DistGNN at world 1 (C3 and C5): time.perf_counter around the
call without synchronising, after warm-up."""
import json
import os
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_2305_17408_b200 import dist as D  # noqa: E402
from paper_2305_17408_b200 import synth  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1)
out = {}
for name in ("C3", "C5"):
    cfg = bench.CONFIGS[name]
    _, rg, dec, net, _ = bench.build_workload(cfg)
    V, dims = cfg["V"], cfg["dims"]
    x = torch.randn((V, dims[0]), device="cuda")
    lab, msk = synth.labels_and_mask(V, dims[-1], seed=0)
    labels = torch.from_numpy(lab).cuda()
    mask = torch.from_numpy(msk).cuda()
    n = int(msk.sum())
    net.autotune()
    dnet = D.DistGNN.build(cfg["model"], dims, dec, 0, 1, subject_t=net.subject_t)
    dnet.autotune()
    xe = dnet.input_ext(x)
    r = {}
    for label, fn in (("gnn", lambda: net.train_step(x, labels, mask, n, 0.0)),
                      ("distgnn", lambda: dnet.train_step(xe, labels, mask, n, 0.0))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        host = []
        dev = []
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            t0 = time.perf_counter()
            fn()
            host.append((time.perf_counter() - t0) * 1e3)
            e.record()
            torch.cuda.synchronize()
            dev.append(s.elapsed_time(e))
        r[label] = {"host_ms": round(sorted(host)[2], 3), "device_ms": round(sorted(dev)[2], 3)}
    out[name] = r
    print(json.dumps(out), flush=True)
dist.destroy_process_group()
