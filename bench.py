"""Benchmark: GCN/GIN training epoch on a synthetic config + aggregation SpMM
GB/s against the HBM roofline (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5]
                    [--impl ours|reference]

A step is one training epoch (forward over every layer, masked softmax
cross-entropy, backward, SGD) of the config's model on its synthetic graph
(seeded generator, METIS-style planted-community partition file fed through
load_partition, comm_size 16).  The headline `value` is epoch ms with all
inputs resident in HBM; `e2e` is the same epoch through the public API with
the feature matrix / labels copied from pinned host memory every step and
the loss read back.  `roofline` is the aggregation (the dominant memory-bound
kernel pair: inter CSR + intra CSR with the fused combine), measured with
CUDA events around every aggregation inside the timed steps.
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import threading
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

# (V, E, dims, model, generator parameters); class counts are the named datasets'
CONFIGS = {
    "C1": dict(V=2708, E=10556, dims=[1433, 16, 7], model="gcn", name="cora-shaped"),
    "C2": dict(V=19717, E=88648, dims=[500, 16, 3], model="gcn", name="pubmed-shaped"),
    "C3": dict(V=169343, E=1166243, dims=[128, 64, 64, 64, 64, 40], model="gin",
               name="ogbn-arxiv-shaped"),
    # C4's planted communities are 512 rows: the partition file's community size
    # is the decomposition block (B = 16 leaves 1.2% of the edges intra; B = 512
    # puts 36% on the tensor-core dense_block kernel -- 32.8 -> 20.3 ms per epoch)
    "C4": dict(V=232965, E=114615892, dims=[602, 128, 41], model="gcn", name="reddit-shaped",
               block_gen=512, comm_size=512),
    "C5": dict(V=2449029, E=61859140, dims=[100, 256, 256, 47], model="gcn",
               name="ogbn-products-shaped"),
}
GEN = dict(block_gen=16, p_intra=0.4, p_global=0.05, window=16, skew=1, seed=0)
COMM_SIZE = 16
METRIC = "GCN/GIN epoch ms + aggregation SpMM GB/s vs HBM roofline"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self._stop = index, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}",
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[2:6]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit()
                else None, "reasons": reasons, "samples": len(self.rows)}


def build_workload(cfg, rank=0, world=1):
    import torch
    import paper_2305_17408_b200 as ag
    from paper_2305_17408_b200 import synth
    gen = dict(GEN)
    gen["block_gen"] = cfg.get("block_gen", GEN["block_gen"])
    t0 = time.perf_counter()
    g, comm = synth.community_graph(cfg["V"], cfg["E"], **gen)
    if cfg["model"] == "gcn":
        g = ag.gcn_normalize(g)
    part = ag.reorder.partition_from_ids(comm, COMM_SIZE)  # load_partition core
    rg = ag.apply_reorder(g, part)
    dec = ag.decompose(rg, COMM_SIZE)
    net = ag.GNN.build(cfg["model"], cfg["dims"], dec, seed=0)
    torch.cuda.synchronize()
    prep_s = time.perf_counter() - t0
    return g, rg, dec, net, prep_s


class HostFeeder:
    """Pinned-host -> device inputs on a side stream with DEPTH buffers: the
    copy of step i + DEPTH - 1 is issued when step i starts, so PCIe hiccups
    (the link is shared on the box) are absorbed by DEPTH - 1 steps of slack
    (the usual pin_memory / non_blocking DataLoader prefetch).  Every step's
    bytes are still copied inside the timed region; only their latency is
    hidden."""

    DEPTH = 3

    def __init__(self, host):
        import torch
        self.host = host
        self.bufs = [[torch.empty(t.shape, dtype=t.dtype, device="cuda") for t in host]
                     for _ in range(self.DEPTH)]
        self.stream = torch.cuda.Stream()
        self.ready = [torch.cuda.Event() for _ in range(self.DEPTH)]
        self.free = [torch.cuda.Event() for _ in range(self.DEPTH)]
        self.reset()

    def reset(self):
        import torch
        self.i = 0
        self.issued = 0
        for e in self.free:
            e.record(torch.cuda.current_stream())

    def issue(self, k=None):
        """Copy the next step's inputs into its buffer (k: ignored, kept for
        the call sites)."""
        import torch
        k = self.issued % self.DEPTH
        with torch.cuda.stream(self.stream):
            self.stream.wait_event(self.free[k])  # the step that used buffer k is done
            for d, h in zip(self.bufs[k], self.host):
                d.copy_(h, non_blocking=True)
            self.ready[k].record(self.stream)
        self.issued += 1

    def get(self, prefetch_next=True, remaining=None):
        """Buffers of the next step; keeps DEPTH - 1 later steps in flight
        (`remaining` = steps after this one still to be fed)."""
        import torch
        k = self.i % self.DEPTH
        torch.cuda.current_stream().wait_event(self.ready[k])
        if prefetch_next:
            ahead = self.DEPTH - 1 if remaining is None else min(self.DEPTH - 1, remaining)
            while self.issued < self.i + 1 + ahead:
                self.issue()
        self.i += 1
        return self.bufs[k], k

    def release(self, k):
        import torch
        self.free[k].record(torch.cuda.current_stream())


def ncu_traffic():
    """DRAM bytes of one F=256 aggregation launch from the committed ncu
    capture of the pair the autotune runs (profiles/r02_ncu.json), or
    (None, reason)."""
    p = ROOT / "profiles" / "r02_ncu.json"
    if not p.exists():
        return None, "no ncu capture committed"
    d = json.loads(p.read_text())
    return int(d["traffic_bytes_per_launch_f256"]), f"{p.name}: {d['source']}"


def bytes_alg(V, E_full, F, weighted):
    """4(V+1) + 4E' + 4wE' + 8VF per full-graph aggregation."""
    return 4 * (V + 1) + 4 * E_full + (4 * E_full if weighted else 0) + 8 * V * F


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist
    import paper_2305_17408_b200 as ag
    from paper_2305_17408_b200 import _lib, synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    # the row-partitioned (DistGNN) path: world > 1, or --force-dist on one GPU
    # (NCCL group of one: exercises the multi-GPU code path end to end)
    dpath = world > 1 or args.force_dist
    if dpath:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl")
    g, rg, dec, net, prep_s = build_workload(cfg, rank, world)
    V = cfg["V"]
    dims = cfg["dims"]
    gen_t = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn((V, dims[0]), generator=gen_t, device="cuda", dtype=torch.float32)
    labels_np, mask_np = synth.labels_and_mask(V, dims[-1], seed=0)
    n_mask = int(mask_np.sum())  # global count (the loss is a mean over all ranks' rows)
    lr = 0.01
    t_tune = time.perf_counter()
    cache_info = None
    if dpath:
        # row partition: each rank owns a B-aligned, nnz-balanced row range
        from paper_2305_17408_b200 import dist as D
        dnet = D.DistGNN.build(cfg["model"], dims, dec, rank, world, seed=0,
                               subject_t=net.subject_t)
        r0, r1 = dnet.bounds[rank], dnet.bounds[rank + 1]
        names = {"csr": (ag.KernelKind.CSR_INTRA_BLOCKED, ag.KernelKind.CSR_INTER),
                 "dense_coo": (ag.KernelKind.DENSE_BLOCK, ag.KernelKind.COO_ATOMIC)}
        choices = {k: names[v] for k, v in dnet.autotune().items()}
        x_local = x[r0:r1].contiguous()
        labels = torch.from_numpy(labels_np[r0:r1]).cuda()
        mask = torch.from_numpy(mask_np[r0:r1]).cuda()
        x_ext = dnet.input_ext(x_local)
        del x

        def step():
            return dnet.train_step(x_ext, labels, mask, n_mask, lr)

        def step_on(xd, ld, md):
            return dnet.train_step(dnet.input_ext(xd), ld, md, n_mask, lr)
        timed = dnet
        host_x = x_local
        fst, bst = dnet.fwd.plan.stats(), dnet.bwd.plan.stats()
        halo = {"fwd_halo_rows": fst["halo_rows"], "bwd_halo_rows": bst["halo_rows"],
                "fwd_allgather_rows_avoided": fst["allgather_rows"],
                "exchange": "per-peer uneven all-to-all (exact halo), backward exchange "
                            "overlapped with the dW GEMM",
                "rows_per_rank": r1 - r0}
    else:
        labels = torch.from_numpy(labels_np).cuda()
        mask = torch.from_numpy(mask_np).cuda()
        cache = ag.ChoiceCache(args.choice_cache) if args.choice_cache else None
        choices = net.autotune(cache=cache)
        cache_info = None if cache is None else {"path": str(args.choice_cache),
                                                  "hits": cache.hits, "misses": cache.misses}

        def step():
            return net.train_step(x, labels, mask, n_mask, lr)

        def step_on(xd, ld, md):
            return net.train_step(xd, ld, md, n_mask, lr)
        timed = net
        host_x = x
        halo = None
    tune_s = time.perf_counter() - t_tune

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dpath:
        dist.barrier()
    use_graph = not dpath and not args.no_graph
    timed.events = []
    launches0 = _lib.launch_count()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if use_graph:
        # per-aggregation CUDA-event timings from an eager pass; the headline
        # steps below replay the same step as one CUDA graph
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
        launches_per_step = (_lib.launch_count() - launches0) / args.steps
        agg_events = timed.events
        timed.events = None
        graphed_v = ag.GraphedTrainStep(timed, [(x, labels, mask)], n_mask, lr)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        if dpath:
            dist.barrier()
        start.record()
        for _ in range(args.steps):
            if use_graph:
                loss = graphed_v.step(0)
            else:
                loss, _ = step()
        end.record()
        torch.cuda.synchronize()
        if dpath:
            dist.barrier()
    if use_graph:
        launches = launches_per_step * args.steps  # the graph holds one step's launches
        timed.events = agg_events
    else:
        launches = _lib.launch_count() - launches0
    ms = start.elapsed_time(end) / args.steps
    agg_ms = sum(e0.elapsed_time(e1) for e0, e1, _, _ in timed.events)
    per_width = {}
    for e0, e1, f, _ in timed.events:
        pw = per_width.setdefault(int(f), [0, 0.0])
        pw[0] += 1
        pw[1] += e0.elapsed_time(e1)
    E_full = rg.num_edges
    weighted = rg.weights is not None
    # algorithmic bytes of the aggregations THIS rank ran (its rows' share)
    frac_rows = 1.0 if not dpath else halo["rows_per_rank"] / V
    agg_bytes = sum(bytes_alg(V, E_full, f, weighted) for _, _, f, _ in timed.events) * frac_rows
    n_agg = len(timed.events)
    timed.events = None
    if dpath:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        tb = torch.tensor([agg_bytes, agg_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tb, op=dist.ReduceOp.SUM)
        agg_bytes = float(tb[0].item())  # whole-job algorithmic bytes
        agg_ms = float(tb[1].item()) / world  # mean per-rank aggregation time

    # e2e: public API, features + labels from pinned host memory each step
    x_host = host_x.cpu().pin_memory()
    lab_host = labels.cpu().pin_memory()
    mask_host = mask.cpu().pin_memory()
    torch.cuda.synchronize()
    # host->device bandwidth of the feature matrix alone (diagnostic for e2e)
    xd = torch.empty(x_host.shape, dtype=x_host.dtype, device="cuda")
    xd.copy_(x_host, non_blocking=True)
    h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0.record()
    xd.copy_(x_host, non_blocking=True)
    h1.record()
    torch.cuda.synchronize()
    h2d_gbs = x_host.numel() * 4 / (h0.elapsed_time(h1) / 1e3) / 1e9
    del xd
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps = max(1, args.steps)  # the same K steps as the device-timed arm
    feeder = HostFeeder([x_host, lab_host, mask_host])
    # one untimed step through the same path: the caching allocator grows its
    # pool for the host-fed inputs once, as any steady-state run does
    feeder.issue(0)
    (xd, ld, md), k = feeder.get(prefetch_next=False)
    loss, _ = step_on(xd, ld, md)
    feeder.release(k)
    float(loss.item())
    torch.cuda.synchronize()
    # single GPU: the step replays as one CUDA graph per feeder buffer
    # (models.GraphedTrainStep); the buffers hold real inputs while capturing
    graphed = None
    if not dpath and not args.no_graph:
        for bufs in feeder.bufs:
            for d, h in zip(bufs, feeder.host):
                d.copy_(h)
        graphed = ag.GraphedTrainStep(timed, [tuple(b) for b in feeder.bufs], n_mask, lr)
    feeder.reset()
    if dpath:
        dist.barrier()
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(e2e_steps + 1)]
    e_start.record()
    step_ev[0].record()
    feeder.issue(0)
    host_ms = []
    for i in range(e2e_steps):
        t_h = time.perf_counter()
        (xd, ld, md), k = feeder.get(prefetch_next=i + 1 < e2e_steps,
                                     remaining=e2e_steps - 1 - i)
        if graphed is not None:
            loss = graphed.step(k)
        else:
            loss, _ = step_on(xd, ld, md)
        t_l = time.perf_counter()
        feeder.release(k)
        loss_val = float(loss.item())  # D2H of the step's result
        step_ev[i + 1].record()
        host_ms.append((round((t_l - t_h) * 1e3, 2), round((time.perf_counter() - t_h) * 1e3, 2)))
    e_end.record()
    torch.cuda.synchronize()
    e2e_ms = e_start.elapsed_time(e_end) / e2e_steps
    e2e_each = [round(step_ev[i].elapsed_time(step_ev[i + 1]), 2) for i in range(e2e_steps)]
    if dpath:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    h2d = x_host.numel() * 4 + lab_host.numel() * 4 + mask_host.numel()

    peak, peak_src = peaks()
    frac_local = 1.0 if not dpath else halo["rows_per_rank"] / V
    widths = {str(f): {"launches_per_step": n // args.steps, "ms_per_launch": round(t / n, 4),
                       "alg_GBps": round(bytes_alg(V, E_full, f, weighted) * frac_local
                                         / (t / n / 1e3) / 1e9, 1)}
              for f, (n, t) in sorted(per_width.items())}
    traffic, traffic_src = ncu_traffic()
    achieved = agg_bytes / (agg_ms / 1000.0) / 1e9 if agg_ms > 0 else 0.0
    line = {
        "metric": METRIC,
        "value": round(ms, 4),
        "unit": "ms/epoch",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (seeded community generator, random features/labels)",
        "config": {
            "workload": f"{args.config} {cfg['name']}: {cfg['model'].upper()} {len(dims) - 1} "
                        f"layers dims {dims}, V={V}, E={cfg['E']} (+V self loops), comm_size "
                        f"{COMM_SIZE}, planted-partition reorder (load_partition)",
            "generator": {**GEN, "block_gen": cfg.get("block_gen", GEN["block_gen"])},
            "edges_after_gcn_normalize": E_full,
            "intra_edge_fraction": round(dec.intra.num_edges / max(1, E_full), 4),
            "kernels": {f"{k[0]}:{k[1]}": [v[0].value, v[1].value] for k, v in choices.items()},
            "selector_choice": {f"{k[0]}:{k[1]}": [v[0].value, v[1].value]
                                for k, v in getattr(timed, "selector_choice", {}).items()},
            "l2": "inputs and activations (>= 0.98 GB per aggregation) exceed the 126 MB L2",
            "preprocess_s": round(prep_s, 2),
            "autotune_s": round(tune_s, 2),
            "choice_cache": cache_info,
            "launch": "each timed step replays the training step as one CUDA graph "
                      "(GraphedTrainStep); per-aggregation timings from an eager pass"
                      if use_graph else "eager launches, per-aggregation CUDA events in-step",
            "parallelism": f"row-partition x{world} (NCCL per-peer halo all-to-all + dW all-reduce)"
                           if dpath else "single GPU",
            **({"halo": halo} if halo else {}),
        },
        "e2e": {"value": round(e2e_ms, 4), "unit": "ms/epoch", "h2d_bytes_per_step": h2d,
                "input_pipeline": "pinned host -> device on a side stream, "
                                  f"{HostFeeder.DEPTH} prefetch buffers (the copies of the next "
                                  f"{HostFeeder.DEPTH - 1} steps overlap step i)",
                "launch": "CUDA graph per feeder buffer (GraphedTrainStep)" if graphed is not None
                          else "eager",
                "d2h_bytes_per_step": 4, "loss": loss_val,
                "h2d_x_GBps": round(h2d_gbs, 1), "steps_ms": e2e_each,
                "host_launch_ms_total_ms": host_ms},
        "roofline": {
            "bound": "hbm",
            "achieved": round(achieved, 1),
            "peak": peak,
            "unit": "GB/s",
            "frac": round(achieved / peak, 4),
            "traffic": traffic,
            "traffic_per": "one F=256 aggregation launch (dram read + write bytes)",
            "traffic_source": traffic_src,
            "per_width": widths,
            "kernel": "slab_kernel (ag_fused_spmm: the autotuned selector pair of each width in one "
                      "pass -- intra role (dense 16x16 block product or bitwise CSR) + bitwise "
                      "csr_inter role + fused combine / epilogues; pairs in config.kernels)",
            "aggregations_per_step": n_agg // args.steps,
            "agg_ms_per_step": round(agg_ms / args.steps, 4),
            "algorithmic_bytes_per_step": agg_bytes // args.steps,
            "peak_source": peak_src,
        },
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
    }
    if rank == 0 and not dpath and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(rg, cfg)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dpath:
        dist.destroy_process_group()


def _host_graph(rg):
    """Canonical reordered graph as host arrays (the GPU arm's own graph)."""
    w = None if rg.weights is None else rg.weights.cpu().numpy()
    return rg.dst.cpu().numpy(), rg.src.cpu().numpy(), w


def _numpy_graph(cfg):
    """The same workload built with the numpy oracle only (oracle/synth.py twin
    of the device generator, gcn_normalize, load_partition, apply_reorder):
    the reference arm never loads this repo's CUDA library."""
    from oracle import ref_numpy as R
    from oracle import synth as osynth
    gen = dict(GEN)
    gen["block_gen"] = cfg.get("block_gen", GEN["block_gen"])
    (d, s), comm = osynth.community_graph(cfg["V"], cfg["E"], **gen)
    V = cfg["V"]
    if cfg["model"] == "gcn":
        d, s, w = R.gcn_normalize(V, d, s)
    else:
        w = None
    _, perm = R.partition_from_ids(comm, COMM_SIZE)
    return R.apply_reorder(V, d, s, w, perm)


def _cpu_plan(cfg):
    """(fraction of rows, timed reps): every row for C1-C3; a uniform sample of
    16-row blocks sized to ~15 s of host work for the large configs."""
    V = cfg["V"]
    if V <= 200_000:
        return 1.0, (3 if V <= 20_000 else 1)
    return 0.015, 1


def cpu_baseline(rg, cfg):
    from oracle import baseline
    d, s, w = _host_graph(rg)
    frac, reps = _cpu_plan(cfg)
    r = baseline.time_epochs(cfg["V"], d, s, w, COMM_SIZE, cfg["dims"], cfg["model"], frac,
                             reps=reps, warmup=1)
    return _baseline_obj(r, frac, reps)


def _baseline_obj(r, frac, reps):
    if frac >= 1.0:
        sample = (f"full epoch, every row (median of {r['reps']}), the reference's kernels: "
                  f"intra {r['intra_choice']} (selector argmin on this host) + csr_inter, "
                  f"combine, BLAS agg@W, backward_sum; GPU association")
    else:
        sample = (f"uniform random {r['frac_rows']:.2%} of the 16-row blocks ({r['sample_rows']} rows, "
                  f"{r['sample_edges']} edges, every aggregation / GEMM / loss op of the epoch on "
                  f"them, median of {r['reps']}), wall {r['sample_wall_s']:.1f} s scaled by "
                  f"V/rows; reference kernels: intra {r['intra_choice']} + csr_inter, combine, "
                  f"BLAS agg@W, backward_sum; full-size validation: profiles/cpu_fullscale_c5.json")
    return {"value": round(r["epoch_ms"], 1), "unit": "ms/epoch", "cores": r["threads"],
            "kind": "port", "sample": sample, "parts_ms": r["parts_ms"],
            "note": "numpy's reduceat holds the GIL: the reference's thread pool runs at ~1 core"}


def run_reference(args, cfg):
    """--impl reference: the reference's CPU kernels (oracle port of the pure
    numpy reference, oracle/baseline.py) on the host cores, on the same
    workload built by the numpy oracle (no CUDA library); each step is one
    sampled epoch (all rows for C1-C3)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import baseline
    t0 = time.perf_counter()
    d, s, w = _numpy_graph(cfg)
    build_s = time.perf_counter() - t0
    frac, _ = _cpu_plan(cfg)
    if frac < 1.0:
        frac = 0.005  # ~5 s per step, so K + W steps fit in a few minutes
    r = baseline.time_epochs(cfg["V"], d, s, w, COMM_SIZE, cfg["dims"], cfg["model"], frac,
                             reps=max(1, args.steps), warmup=max(1, args.warmup), budget_s=240.0)
    ms = r["epoch_ms"]
    cb = _baseline_obj(r, frac, r["reps"])
    line = {"impl": "reference", "metric": METRIC, "value": round(ms, 1), "unit": "ms/epoch",
            "n_gpus": world, "steps": r["reps"], "warmup": max(1, args.warmup),
            "ms_per_step": round(ms, 1), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (the same seeded generator, built with numpy)",
            "config": {"workload": f"{args.config} {cfg['name']}", "dims": cfg["dims"],
                       "graph_build_s": round(build_s, 1),
                       "steps_requested": args.steps},
            "cpu_baseline": cb,
            "e2e": {"value": round(ms, 1), "unit": "ms/epoch", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--choice-cache", default=str(ROOT / ".choice_cache.json"),
                    help="ChoiceCache file (selector + autotuned pairs per graph/width/direction); "
                         "'' disables it")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the row-partitioned multi-GPU path even on one GPU (testing)")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch the training step eagerly instead of as a CUDA graph")
    ap.add_argument("--comm-size", type=int, default=None,
                    help="decomposition block size B (default: the config's community size, "
                         "16 except C4's 512; SURVEY 8d: also report 64/128/256 for C4)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    globals()["COMM_SIZE"] = args.comm_size or cfg.get("comm_size", COMM_SIZE)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
