"""Per-kernel device time of one C5 training step (torch.profiler / CUPTI).

    python scripts/step_profile.py [--config C5] [--steps 3]
"""
import argparse
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2305_17408_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    g, rg, dec, net, prep = bench.build_workload(cfg)
    V, dims = cfg["V"], cfg["dims"]
    x = torch.randn((V, dims[0]), device="cuda")
    labels_np, mask_np = synth.labels_and_mask(V, dims[-1], seed=0)
    labels = torch.from_numpy(labels_np).cuda()
    mask = torch.from_numpy(mask_np).cuda()
    n_mask = int(mask_np.sum())
    kernels = net.autotune()
    for _ in range(3):
        net.train_step(x, labels, mask, n_mask, 0.01)
    torch.cuda.synchronize()
    acts = [torch.profiler.ProfilerActivity.CUDA]
    with torch.profiler.profile(activities=acts) as prof:
        for _ in range(args.steps):
            net.train_step(x, labels, mask, n_mask, 0.01)
        torch.cuda.synchronize()
    per = defaultdict(lambda: [0, 0.0])
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            name = ev.name
            for key in ("slab_kernel", "tc_gemm_kernel", "splitk_sum", "xent", "sgd", "tf32_split",
                        "Memset", "Memcpy"):
                if key in name:
                    name = key + (name[name.find("<"):name.find(">") + 1] if "<" in name else "")
                    break
            per[name][0] += 1
            per[name][1] += ev.device_time_total / 1000.0
    rows = sorted(per.items(), key=lambda kv: -kv[1][1])
    total = sum(v[1] for v in per.values()) / args.steps
    out = {"config": args.config, "kernels": {str(k): str(v) for k, v in kernels.items()},
           "step_ms_sum_of_kernels": round(total, 3),
           "per_kernel_ms_per_step": {k: [v[0] // args.steps, round(v[1] / args.steps, 3)]
                                      for k, v in rows}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
