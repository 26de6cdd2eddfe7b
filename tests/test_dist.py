"""Multi-GPU host logic on CPU: world-size-2 and -4 gloo processes run the real
partition / peer-set / remap / all-to-all code of paper_2305_17408_b200.dist
on CPU tensors, with the oracle's numpy CSR aggregation standing in for the
device kernel.  Every rank's local aggregation over its halo-extended features
must be BITWISE equal to its rows of the global aggregation,
and the bucketed dW all-reduce must sum the per-rank partial GEMMs."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from oracle import ref_numpy as R  # noqa: E402
from paper_2305_17408_b200 import dist as D  # noqa: E402


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _graph(seed=0, V=700, E=6000, B=16, weighted=True):
    rng = np.random.default_rng(seed)
    # community-local graph so the halo is a small part of each rank
    d = rng.integers(0, V, E)
    off = rng.integers(-40, 41, E)
    s = np.clip(d + off, 0, V - 1)
    keep = s != d
    d, s = d[keep], s[keep]
    d, s, w = R.canonical(V, d, s, rng.uniform(0.1, 2.0, d.size).astype(np.float32)
                          if weighted else None)
    if w is None:
        w = np.ones(d.size, np.float32)
    rp, col, val = R.to_csr(V, d, s, w)
    return V, rp, col, val


def _role_layout(V, rp, col, val, B):
    """Role-ordered copy (intra run first, then the inter edges) in numpy."""
    rcol, rval, mid = np.empty_like(col), np.empty_like(val), np.empty(V, np.int64)
    for r in range(V):
        s, e = rp[r], rp[r + 1]
        c = col[s:e]
        cb = (r // B) * B
        ia, ib = np.searchsorted(c, cb), np.searchsorted(c, cb + B)
        order = np.r_[np.arange(ia, ib), np.arange(0, ia), np.arange(ib, e - s)]
        rcol[s:e], rval[s:e] = c[order], val[s:e][order]
        mid[r] = s + (ib - ia)
    return rcol, rval, mid


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, F = 16, 6
        V, rp, col, val = _graph()
        x = np.random.default_rng(1).standard_normal((V, F)).astype(np.float32)
        ref = R.csr_aggregate(V, rp, col, val, x, "sum")[0]
        t_rp, t_col, t_val = (torch.from_numpy(np.ascontiguousarray(a)) for a in (rp, col, val))
        bounds = D.balanced_bounds(t_rp, world, B)
        assert all(b % B == 0 for b in bounds[:-1]) and bounds[-1] == V
        op = D.LocalOperator.build(t_rp, t_col, t_val, bounds, rank, B)
        plan = op.plan
        r0, r1 = bounds[rank], bounds[rank + 1]
        x_ext = plan.new_ext(F, "cpu")
        x_ext.zero_()
        x_ext[:plan.n_local] = torch.from_numpy(x[r0:r1])
        plan.exchange(x_ext)
        lrp = op.row_ptr.numpy().astype(np.int64)
        got = R.csr_aggregate(plan.n_local, lrp, op.col.numpy().astype(np.int64),
                              op.val.numpy(), x_ext.numpy(), "sum")[0]
        bitwise = bool(np.array_equal(got.view(np.uint32), ref[r0:r1].view(np.uint32)))
        # role-ordered operator: remapped columns map back to the global ones
        rcol, rval, mid = _role_layout(V, rp, col, val, B)
        rop = D.LocalOperator.build(t_rp, t_col, t_val, bounds, rank, B,
                                    mid=torch.from_numpy(mid), role_col=torch.from_numpy(rcol),
                                    role_val=torch.from_numpy(rval))
        ext_to_global = np.full(plan.ext_rows, -1, np.int64)
        ext_to_global[:plan.n_local] = np.arange(r0, r1)
        for j, S in enumerate(plan.recv_sets):
            base = plan.halo_base + plan.recv_offsets[j]
            ext_to_global[base:base + S.numel()] = S.numpy()
        # exact halo: every received row is referenced by this rank's edges
        lcol = op.col.numpy().astype(np.int64)
        used = np.unique(lcol[lcol >= plan.halo_base])
        exact = bool(used.size == plan.ext_rows - plan.halo_base
                     and np.array_equal(x_ext.numpy()[plan.halo_base:],
                                        x[ext_to_global[plan.halo_base:]]))
        e0, e1 = rp[r0], rp[r1]
        role_ok = bool(np.array_equal(ext_to_global[rop.col.numpy()], rcol[e0:e1])
                       and np.array_equal(rop.mid.numpy() + e0, mid[r0:r1]))
        # bucketed dW all-reduce == the GEMM over all rows
        g = np.random.default_rng(2).standard_normal((V, 3)).astype(np.float32)
        part = torch.from_numpy(x[r0:r1].T.astype(np.float64) @ g[r0:r1].astype(np.float64))
        dist.all_reduce(part)
        dw_ok = bool(np.allclose(part.numpy(), x.T.astype(np.float64) @ g.astype(np.float64),
                                 rtol=1e-12, atol=1e-12))
        st = plan.stats()
        halo_frac = st["halo_rows"] / max(1, plan.n_local)
        out[rank] = (bitwise, role_ok, dw_ok, plan.n_local, halo_frac, exact,
                     st["halo_rows"] <= st["allgather_rows"])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_row_partition_halo_exchange_gloo(world):
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert sorted(out.keys()) == list(range(world))
    for rank in range(world):
        bitwise, role_ok, dw_ok, n_local, halo_frac, exact, leq = out[rank]
        assert bitwise, f"rank {rank}: local aggregation differs from the global rows"
        assert exact, f"rank {rank}: the halo holds rows nobody references, or wrong rows"
        assert leq, f"rank {rank}: per-peer halo larger than the padded all-gather"
        assert role_ok, f"rank {rank}: role-ordered remap"
        assert dw_ok, f"rank {rank}: dW all-reduce"
        assert n_local > 0 and halo_frac < 0.5


def test_balanced_bounds_properties():
    rp = torch.tensor([0, 5, 5, 9, 30, 31, 40, 41, 41, 60, 61, 61, 70, 72, 80, 90, 91, 100])
    for world in (1, 2, 3, 4):
        b = D.balanced_bounds(rp, world, 4)
        assert b[0] == 0 and b[-1] == 17 and len(b) == world + 1
        assert all(x <= y for x, y in zip(b, b[1:]))
        assert all(x % 4 == 0 for x in b[:-1])


def test_send_sets_and_remap_single_process():
    V, rp, col, val = _graph(V=300, E=2000)
    t_rp, t_col = torch.from_numpy(rp), torch.from_numpy(col)
    bounds = D.balanced_bounds(t_rp, 3, 16)
    sets = D.send_sets(t_rp, t_col, bounds)
    # brute force
    own = np.searchsorted(np.array(bounds[1:-1]), np.arange(V), side="right")
    dst = np.repeat(np.arange(V), np.diff(rp))
    for j in range(3):
        want = np.unique(col[(own[col] == j) & (own[dst] != j)])
        assert np.array_equal(sets[j].numpy(), want)
    plan = D.HaloPlan.build(t_rp, t_col, bounds, 1, 16)
    r0, r1 = bounds[1], bounds[2]
    cols = col[rp[r0]:rp[r1]]
    m = plan.remap(torch.from_numpy(cols)).numpy()
    assert m.min() >= 0 and m.max() < plan.ext_rows
    local = (cols >= r0) & (cols < r1)
    assert np.array_equal(m[local], cols[local] - r0)
    assert (m[~local] >= plan.halo_base).all()
