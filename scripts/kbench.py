"""Per-kernel timing on a bench config (CUDA events, warm), for development.

    python scripts/kbench.py [--config C5] [--feat 256]
"""
import argparse
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2305_17408_b200 as ag  # noqa: E402
from paper_2305_17408_b200 import kernels as K  # noqa: E402
from paper_2305_17408_b200.decompose import full_graph  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--feat", type=int, nargs="+", default=[256, 100])
    ap.add_argument("--only", default=None, help="run just this kernel once (for ncu)")
    ap.add_argument("--pair", default="csr_intra_blocked,csr_inter",
                    help="intra,inter kernel pair of --only fused_pair / --suite agg")
    ap.add_argument("--suite", default="all", help="all | agg (fused aggregation pairs only)")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    g, rg, dec, net, prep = bench.build_workload(cfg)
    V = cfg["V"]
    E = rg.num_edges
    out = {"V": V, "E": E, "intra": dec.intra.num_edges, "prep_s": prep}
    intra, inter = K.decomposed_execs(dec)
    full = K.to_csr(full_graph(dec))
    lens = (full.row_ptr[1:] - full.row_ptr[:-1]).float()
    out["deg_mean"] = float(lens.mean())
    out["deg_max"] = float(lens.max())
    out["rows_over_128"] = int((lens > 128).sum())
    for F in args.feat:
        x = torch.randn((V, F), device="cuda")
        y = torch.empty_like(x)
        if args.only == "gemm":
            w = torch.randn((F, 256), device="cuda")
            K.gemm(x, w)
            torch.cuda.synchronize()
            continue
        ki, ke = (ag.KernelKind(k) for k in args.pair.split(","))
        if args.only == "gemm_dw":
            g256 = torch.randn((V, 256), device="cuda")
            K.gemm(x, g256, trans_a=True)
            torch.cuda.synchronize()
            continue
        if args.only == "gemm_dh48":
            q48 = torch.randn((V, 48), device="cuda")
            w48 = torch.randn((256, 48), device="cuda")
            mk = torch.randn((V, 256), device="cuda")
            K.gemm(q48, w48, trans_b=True, relu_mask=mk)
            torch.cuda.synchronize()
            continue
        if args.only == "fused_pair":
            K.run_fused_pair(dec, x, y, ag.AggregateOp.SUM, kernel_intra=ki, kernel_inter=ke)
            torch.cuda.synchronize()
            continue
        if args.suite == "gemm":
            if F != args.feat[0]:
                continue
            g256 = torch.randn((V, 256), device="cuda")
            h256 = torch.randn((V, 256), device="cuda")
            x100 = torch.randn((V, 100), device="cuda")
            q48 = torch.randn((V, 48), device="cuda")
            w100 = torch.randn((100, 256), device="cuda")
            w256 = torch.randn((256, 256), device="cuda")
            w48 = torch.randn((256, 48), device="cuda")
            shapes = {
                "fwd_100x256": lambda: K.gemm(x100, w100),
                "fwd_256x256": lambda: K.gemm(h256, w256),
                "fwd_256x48": lambda: K.gemm(h256, w48),
                "dW_256x48": lambda: K.gemm(h256, q48, trans_a=True),
                "dH_48x256_mask": lambda: K.gemm(q48, w48, trans_b=True, relu_mask=h256),
                "dW_256x256": lambda: K.gemm(h256, g256, trans_a=True),
                "dH_256x256": lambda: K.gemm(g256, w256, trans_b=True),
                "dW_100x256": lambda: K.gemm(x100, g256, trans_a=True),
            }
            res = {k: timeit(fn) for k, fn in shapes.items()}
            import os
            if os.environ.get("KB_GEMM_EXP"):
                for ex in os.environ["KB_GEMM_EXP"].split(","):
                    os.environ["AG_TC_EXP"] = ex
                    for k in ("dH_48x256_mask", "fwd_256x256", "fwd_100x256"):
                        res[f"{k}[exp{ex}]"] = timeit(shapes[k])
                os.environ.pop("AG_TC_EXP")
            ref = h256[:4096].double() @ w256.double()
            got = K.gemm(h256, w256)[:4096].double()
            out["gemm_relerr"] = float(((got - ref).abs() / ref.abs().clamp(min=1.0)).max())
            out["gemm_ms"] = {k: round(v, 4) for k, v in res.items()}
            out["gemm_total_ms"] = round(sum(res.values()), 3)
            continue
        if args.suite == "agg":
            ba = bench.bytes_alg(V, E, F, rg.weights is not None)
            ref = torch.empty_like(x)
            K.run_fused_pair(dec, x, ref, ag.AggregateOp.SUM)
            refd = ref.double()
            res, err = {}, {}
            hrelu = torch.randn_like(x)
            for pki in (ag.KernelKind.CSR_INTRA_BLOCKED, ag.KernelKind.DENSE_BLOCK):
                for pke in (ag.KernelKind.CSR_INTER, ag.KernelKind.COO_ATOMIC):
                    name = f"{pki.value}+{pke.value}"
                    run = lambda d=dec, **kw: K.run_fused_pair(d, x, y, ag.AggregateOp.SUM,
                                                               kernel_intra=pki,
                                                               kernel_inter=pke, **kw)
                    res[name] = timeit(run)
                    err[name] = float(((y.double() - refd).abs()
                                       / refd.abs().clamp(min=1.0)).max())
                    res[name + ":bwd_relu"] = timeit(lambda: run(net.subject_t,
                                                                 relu_src=hrelu))
            gbs = {k: round(ba / (v / 1e3) / 1e9, 1) for k, v in res.items()}
            out[f"F{F}"] = {"ms": {k: round(v, 4) for k, v in res.items()}, "alg_GBps": gbs,
                            "max_rel_vs_bitwise_pair": err, "bytes_alg": ba}
            continue
        ba = bench.bytes_alg(V, E, F, rg.weights is not None)
        res = {}
        import os
        ref = torch.empty_like(x)
        K.run_fused_pair(dec, x, ref, ag.AggregateOp.SUM)
        for vec, notma in (("1", "0"), ("2", "0"), ("2", "1")):
            os.environ["AG_SLAB_VEC"], os.environ["AG_SLAB_NO_TMA"] = vec, notma
            res[f"fused_pair_vec{vec}_notma{notma}"] = timeit(
                lambda: K.run_fused_pair(dec, x, y, ag.AggregateOp.SUM))
            out.setdefault("bitwise_same", []).append(bool(torch.equal(y, ref)))
        os.environ["AG_SLAB_VEC"], os.environ["AG_SLAB_NO_TMA"] = "2", "0"
        os.environ["AG_SLAB_DEBUG"] = "1"
        res["fused_pair_noreduce"] = timeit(lambda: K.run_fused_pair(dec, x, y, ag.AggregateOp.SUM))
        os.environ["AG_SLAB_DEBUG"] = "0"
        out[f"window_F{F}"] = K.to_csr(full_graph(dec)).window()
        res["fused_pair"] = timeit(lambda: K.run_fused_pair(dec, x, y, ag.AggregateOp.SUM))
        res["fused_pair_dense"] = timeit(lambda: K.run_fused_pair(dec, x, y, ag.AggregateOp.SUM,
                                                                 dense_intra=True))
        dect = net.subject_t
        hrelu = torch.randn_like(x)
        res["bwd_pair"] = timeit(lambda: K.run_fused_pair(dect, x, y, ag.AggregateOp.SUM))
        res["bwd_pair_relu"] = timeit(lambda: K.run_fused_pair(dect, x, y, ag.AggregateOp.SUM,
                                                               relu_src=hrelu))
        res["fwd_pair_relu"] = timeit(lambda: K.run_fused_pair(dec, x, y, ag.AggregateOp.SUM,
                                                               relu_src=hrelu))
        out[f"bwd_window_F{F}"] = K.to_csr(full_graph(dect)).window()
        res["fused_full_O1"] = timeit(lambda: K.launch_fused(full, x, y, ag.AggregateOp.SUM))
        res["inter_csr_fused_raw"] = timeit(lambda: K.launch_fused(inter.csr, x, y,
                                                                   ag.AggregateOp.SUM))
        res["intra_csr_fused"] = timeit(lambda: K.launch_fused(intra.csr, x, y,
                                                               ag.AggregateOp.SUM))
        res["inter_coo"] = timeit(lambda: (K.coo_init(y, ag.AggregateOp.SUM),
                                           K.launch_coo(inter.coo, x, y, ag.AggregateOp.SUM)))
        res["intra_dense_block"] = timeit(lambda: K.launch_dense_block(intra.blocks, x, y,
                                                                       ag.AggregateOp.SUM))
        res["full_csr_old"] = timeit(lambda: K.launch_csr(full, x, y, ag.AggregateOp.SUM))
        yo = torch.empty_like(x)
        K.launch_fused(full, x, yo, ag.AggregateOp.SUM)
        out.setdefault("fused_O1_equals_old_csr", []).append(bool(torch.equal(y, yo)))
        res["copy_xy"] = timeit(lambda: y.copy_(x))
        w = torch.randn((F, 256), device="cuda")
        g256 = torch.randn((V, 256), device="cuda")
        for bn in ("256", "128"):
            os.environ["AG_TC_BN"] = bn
            res[f"gemm_Fx256_bn{bn}"] = timeit(lambda: K.gemm(x, w))
            res[f"gemm_dW_bn{bn}"] = timeit(lambda: K.gemm(x, g256, trans_a=True))
            res[f"gemm_dH_bn{bn}"] = timeit(lambda: K.gemm(g256, w, trans_b=True))
        os.environ.pop("AG_TC_BN")
        ref_g = K.gemm(x, w)
        os.environ["AG_TC_RAWHI"] = "1"
        res["gemm_Fx256_rawhi"] = timeit(lambda: K.gemm(x, w))
        res["gemm_dW_rawhi"] = timeit(lambda: K.gemm(x, g256, trans_a=True))
        res["gemm_dH_rawhi"] = timeit(lambda: K.gemm(g256, w, trans_b=True))
        out.setdefault("rawhi_bitwise", []).append(bool(torch.equal(K.gemm(x, w), ref_g)))
        os.environ.pop("AG_TC_RAWHI")
        q48 = torch.randn((V, 48), device="cuda")
        w48 = torch.randn((256, 48), device="cuda")
        mk = torch.randn((V, 256), device="cuda")
        x100 = torch.randn((V, 100), device="cuda")
        w100 = torch.randn((100, 256), device="cuda")
        for bn in ("256", "128"):
            os.environ["AG_TC_BN"] = bn
            res[f"gemm_dH48_mask_bn{bn}"] = timeit(lambda: K.gemm(q48, w48, trans_b=True,
                                                                  relu_mask=mk))
            res[f"gemm_fwd100_bn{bn}"] = timeit(lambda: K.gemm(x100, w100))
        os.environ.pop("AG_TC_BN")
        del q48, mk, x100
        os.environ["AG_TC_EXP"] = "7"
        res["gemm_Fx256_exp7"] = timeit(lambda: K.gemm(x, w))
        os.environ.pop("AG_TC_EXP")
        os.environ["AG_TC_CL"] = "1"
        res["gemm_Fx256_cl1"] = timeit(lambda: K.gemm(x, w))
        res["gemm_dW_cl1"] = timeit(lambda: K.gemm(x, g256, trans_a=True))
        res["gemm_dH_cl1"] = timeit(lambda: K.gemm(g256, w, trans_b=True))
        os.environ.pop("AG_TC_CL")
        ref64 = x.double() @ w.double()
        def relerr(t):
            return float(((t.double() - ref64).abs() / ref64.abs().clamp(min=1.0)).max())
        out.setdefault("gemm_relerr_twoacc", []).append(relerr(K.gemm(x, w)))
        os.environ["AG_TC_ONEACC"] = "1"
        out.setdefault("gemm_relerr_oneacc", []).append(relerr(K.gemm(x, w)))
        res["gemm_Fx256_oneacc"] = timeit(lambda: K.gemm(x, w))
        res["gemm_dW_oneacc"] = timeit(lambda: K.gemm(x, g256, trans_a=True))
        res["gemm_dH_oneacc"] = timeit(lambda: K.gemm(g256, w, trans_b=True))
        os.environ.pop("AG_TC_ONEACC")
        del ref64
        res["gemm_Fx256_simt"] = timeit(lambda: K.gemm(x, w, engine="simt"))
        gbs = {k: round(ba / (v / 1e3) / 1e9, 1) for k, v in res.items() if "gemm" not in k}
        out[f"F{F}"] = {"ms": {k: round(v, 4) for k, v in res.items()}, "alg_GBps": gbs,
                        "bytes_alg": ba}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
