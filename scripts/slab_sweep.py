"""Slab-kernel knob sweep on a bench config (development): every fused pair at
the given widths, forward and backward-with-ReLU-mask, under each setting of
the environment knobs the launcher reads per launch.

    python scripts/slab_sweep.py [--config C5] [--feat 256 100 48]
        [--knob AG_SLAB_CSLEEP=0,100,400]
"""
import argparse
import json
import os
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2305_17408_b200 as ag  # noqa: E402
from paper_2305_17408_b200 import kernels as K  # noqa: E402

PAIRS = [("csr_intra_blocked", "csr_inter"), ("dense_block", "csr_inter"),
         ("csr_intra_blocked", "coo_atomic"), ("dense_block", "coo_atomic")]


def timeit(fn, reps=7):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return sorted(ts)[reps // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--feat", type=int, nargs="+", default=[256, 100, 48])
    ap.add_argument("--knob", action="append", default=[])
    ap.add_argument("--pairs", default="all")
    ap.add_argument("--relu-bits", action="store_true", help="time the bwd pass with a bit mask")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    _, rg, dec, net, _ = bench.build_workload(cfg)
    V, E = cfg["V"], rg.num_edges
    knobs = [(k.split("=")[0], k.split("=")[1].split(",")) for k in args.knob] or [("", [""])]
    pairs = PAIRS if args.pairs == "all" else [tuple(p.split("+")) for p in args.pairs.split(";")]
    from paper_2305_17408_b200.decompose import full_graph
    csr = K.to_csr(full_graph(dec))
    tcsr = K.to_csr(full_graph(net.subject_t))
    out = {"V": V, "E": E, "window": csr.window(), "window_T": tcsr.window(), "results": []}
    print(json.dumps({k: v for k, v in out.items() if k != "results"}), flush=True)
    for F in args.feat:
        x = torch.randn((V, F), device="cuda")
        y = torch.empty_like(x)
        h = torch.randn_like(x)
        ba = bench.bytes_alg(V, E, F, rg.weights is not None)
        for name, vals in knobs:
            for v in vals:
                if name:
                    os.environ[name] = v
                for pi, pe in pairs:
                    ki, ke = ag.KernelKind(pi), ag.KernelKind(pe)
                    fwd = timeit(lambda: K.run_fused_pair(dec, x, y, ag.AggregateOp.SUM,
                                                          kernel_intra=ki, kernel_inter=ke))
                    bwd = timeit(lambda: K.run_fused_pair(net.subject_t, x, y, ag.AggregateOp.SUM,
                                                          kernel_intra=ki, kernel_inter=ke,
                                                          relu_src=h))
                    r = {"F": F, "knob": f"{name}={v}" if name else "", "pair": f"{pi}+{pe}",
                         "fwd_ms": round(fwd, 4), "bwd_relu_ms": round(bwd, 4),
                         "fwd_alg_GBps": round(ba / fwd / 1e6, 1)}
                    out["results"].append(r)
                    print(json.dumps(r), flush=True)
            if name:
                os.environ.pop(name, None)


if __name__ == "__main__":
    main()
