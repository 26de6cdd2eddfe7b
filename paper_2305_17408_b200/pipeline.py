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


@dataclass
class PreparedRun:
    graph: Graph
    decomposed: DecomposedGraph
    reorder_ms: float
    decompose_ms: float


def build_graph(cfg: RunConfig) -> Graph:
    """The edge-list source of the reference (bench.py:103-107); the RMAT /
    planted generators do not scale to the benchmark shapes:
    use paper_2305_17408_b200.synth for synthetic graphs."""
    if cfg.graph_path is not None:
        return load_edge_list(cfg.graph_path)
    raise ValueError("build_graph needs graph_path here; synthetic graphs come from "
                     "paper_2305_17408_b200.synth.community_graph")


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
