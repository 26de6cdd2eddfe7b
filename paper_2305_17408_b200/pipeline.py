"""The preprocessing entry point of the reference harness (bench.py:60-151):
`RunConfig` (its graph-source / reorder / model fields) and `prepare`, which
normalises (GCN), reorders (bfs | none | file:PATH) and decomposes one graph,
timing the stages.  Everything it calls is this package's device path; the
timings bracket the device work with a synchronize, so they are wall times of
finished stages like the reference's perf_counter pairs."""
from __future__ import annotations

import time
from dataclasses import dataclass

import torch

from .decompose import DecomposedGraph, decompose
from .generators import generate_planted_partition, generate_rmat
from .graph import Graph, load_edge_list
from .kernels import AggregateOp
from .models import gcn_normalize
from .reorder import apply_reorder, cluster_bfs, identity_partition, load_partition

MODES = ("O1", "O2", "O3")


@dataclass
class RunConfig:
    """Reference RunConfig (bench.py:60-91): same fields, defaults and checks."""

    graph_path: str | None = None
    rmat: tuple[int, int] | None = None
    planted: tuple[int, int, float, float] | None = None
    comm_size: int = 16
    reorder: str = "bfs"  # bfs | none | file:PATH
    mode: str = "O3"
    op: str = "sum"
    model: str = "agg_only"
    feat_dim: int = 32
    iters: int = 50
    profile_iters: int = 3
    seed: int = 0
    threads: int = 1
    out: str | None = None
    fmt: str = "json"

    def __post_init__(self):
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")
        sources = sum(x is not None for x in (self.graph_path, self.rmat, self.planted))
        if sources > 1:
            raise ValueError("give at most one of graph/rmat/planted")

    def aggregate_op(self) -> AggregateOp:
        return AggregateOp(self.op)

    def as_dict(self) -> dict:
        """The report's `config` object (bench.py:86-101), same keys and order."""
        return {"graph": self.graph_path,
                "rmat": list(self.rmat) if self.rmat else None,
                "planted": list(self.planted) if self.planted else None,
                "comm_size": self.comm_size, "reorder": self.reorder, "mode": self.mode,
                "op": self.op, "model": self.model, "feat_dim": self.feat_dim,
                "iters": self.iters, "profile_iters": self.profile_iters, "seed": self.seed,
                "threads": self.threads}


@dataclass
class PreparedRun:
    graph: Graph
    decomposed: DecomposedGraph
    reorder_ms: float
    decompose_ms: float


def build_graph(cfg: RunConfig) -> Graph:
    """The graph source of a run (bench.py:104-117): edge-list file, RMAT,
    planted partition, or by default a planted graph of 8 groups of
    comm_size vertices (p_in 0.5, p_out 0.01).  The generators are the
    reference's, seed for seed; benchmark-scale synthetic graphs come from
    paper_2305_17408_b200.synth.community_graph."""
    if cfg.graph_path is not None:
        return load_edge_list(cfg.graph_path)
    if cfg.rmat is not None:
        v, e = cfg.rmat
        return generate_rmat(v, e, seed=cfg.seed)
    if cfg.planted is not None:
        groups, size, p_in, p_out = cfg.planted
        return generate_planted_partition(int(groups), int(size), p_in, p_out, seed=cfg.seed)[0]
    return generate_planted_partition(8, cfg.comm_size, 0.5, 0.01, seed=cfg.seed)[0]


def prepare(cfg: RunConfig, graph: Graph) -> PreparedRun:
    """Normalize (GCN), reorder, and decompose one input graph, timing the
    preprocessing stages (bench.py:128-151)."""
    if cfg.model == "gcn":
        graph = gcn_normalize(graph)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if cfg.reorder == "bfs":
        part = cluster_bfs(graph, cfg.comm_size, seed=cfg.seed)
    elif cfg.reorder == "none":
        part = identity_partition(graph.num_vertices, cfg.comm_size)
    elif cfg.reorder.startswith("file:"):
        part = load_partition(cfg.reorder[len("file:"):], cfg.comm_size)
    else:
        raise ValueError(f"unknown reorder method {cfg.reorder!r}")
    reordered = apply_reorder(graph, part)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    d = decompose(reordered, cfg.comm_size)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return PreparedRun(graph=reordered, decomposed=d, reorder_ms=(t1 - t0) * 1000.0,
                       decompose_ms=(t2 - t1) * 1000.0)
