"""The multi-GPU device path on one GPU: G "virtual ranks" built by
paper_2305_17408_b200.dist, their halos filled by indexing the global
features (what the all-gather delivers), aggregated by the real sm_100a fused
kernel.  Each rank's rows must be BITWISE equal to the 1-GPU fused
aggregation, forward and transposed, with the GIN and fused
ReLU-mask epilogues; a world-size-1 DistGNN step must equal GNN.train_step."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2305_17408_b200 as ag  # noqa: E402
from paper_2305_17408_b200 import dist as D  # noqa: E402
from paper_2305_17408_b200 import kernels as K  # noqa: E402
from paper_2305_17408_b200.decompose import full_graph  # noqa: E402
from conftest import rel_error, to_np  # noqa: E402

pytestmark = pytest.mark.gpu


def _setup(model="gcn", V=5000, E=60000, B=16, seed=0):
    from paper_2305_17408_b200 import synth
    g, comm = synth.community_graph(V, E, block_gen=B, p_intra=0.4, p_global=0.02, window=4,
                                    seed=seed)
    if model == "gcn":
        g = ag.gcn_normalize(g)
    rg = ag.apply_reorder(g, ag.reorder.partition_from_ids(comm, B))
    return rg, ag.decompose(rg, B)


def _fill_halo(plan, x_ext, x_global):
    r0 = plan.bounds[plan.rank]
    x_ext[:plan.n_local] = x_global[r0:r0 + plan.n_local]
    for j, S in enumerate(plan.recv_sets):
        base = plan.halo_base + plan.recv_offsets[j]
        x_ext[base:base + S.numel()] = x_global[S]


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("model", ["gcn", "gin"])
def test_virtual_ranks_bitwise(world, model):
    rg, dec = _setup(model)
    B = dec.block_size
    F = 64
    x = torch.randn((rg.num_vertices, F), device="cuda")
    h = torch.randn((rg.num_vertices, F), device="cuda")
    gin = 1.25 if model == "gin" else None
    csr = K.to_csr(full_graph(dec))
    mid, rcol, rval = csr.role_layout(B)
    want = torch.empty_like(x)
    K.run_fused_pair(dec, x, want, ag.AggregateOp.SUM, gin, relu_src=h)
    bounds = D.balanced_bounds(csr.row_ptr, world, B)
    net = D.DistGNN.__new__(D.DistGNN)
    net.model, net.gin_eps, net.events = model, 0.25, None
    net.kernels, net.default_pair, net._dense = {}, "csr", {}
    for rank in range(world):
        op = D.LocalOperator.build(csr.row_ptr, csr.col_idx, csr.kernel_val, bounds, rank, B,
                                   mid=mid, role_col=rcol, role_val=rval,
                                   deg=dec.full_in_degree)
        net.fwd = op
        x_ext = op.plan.new_ext(F, "cuda")
        _fill_halo(op.plan, x_ext, x)
        r0, r1 = bounds[rank], bounds[rank + 1]
        got = net.aggregate(op, x_ext, relu_src=h[r0:r1].contiguous())
        assert torch.equal(got, want[r0:r1]), (world, rank)


class ThreadComm:
    """In-process collectives for G DistGNN "ranks" run as threads on one GPU:
    the uneven all-to-all and the all-reduce through shared tensors, ordered
    by barriers (every rank enqueues on the same CUDA stream, so a peer's
    buffer is complete before the copy that reads it)."""

    def __init__(self, rank, world, shared, barrier):
        self.rank, self.world, self.shared, self.barrier = rank, world, shared, barrier

    def exchange(self, plan, x_ext, async_op=False):
        self.shared[("send", self.rank)] = (x_ext.index_select(0, plan.send_local),
                                            list(plan.send_counts))
        self.barrier.wait()
        off = plan.halo_base
        for j in range(self.world):
            if j == self.rank:
                continue
            buf, counts = self.shared[("send", j)]
            start = sum(counts[:self.rank])
            n = counts[self.rank]
            assert n == plan.recv_counts[j]
            x_ext[off:off + n] = buf[start:start + n]
            off += n
        self.barrier.wait()

        class _Done:
            def wait(self):
                pass
        return _Done() if async_op else None

    def all_reduce(self, t, op=None):
        self.shared[("red", self.rank)] = t.clone()
        self.barrier.wait()
        parts = [self.shared[("red", j)] for j in range(self.world)]
        acc = parts[0].clone()
        for p in parts[1:]:
            acc = torch.maximum(acc, p) if op is not None else acc + p
        self.barrier.wait()
        t.copy_(acc)


def _labels_mask(V, C, seed=5):
    rng = np.random.default_rng(seed)
    labels = torch.from_numpy(rng.integers(0, C, V).astype(np.int32)).cuda()
    mask = torch.from_numpy(rng.random(V) < 0.5).cuda()
    return labels, mask


@pytest.mark.parametrize("model", ["gcn", "gin"])
@pytest.mark.parametrize("pair", ["csr", "dense_coo"])
def test_world1_distgnn_equals_gnn(model, pair):
    """One rank: the reassociated DistGNN step equals GNN.train_step (same
    association, same fused pair)."""
    rg, dec = _setup(model, V=3000, E=30000)
    dims = [32, 24, 16, 5]
    ref = ag.GNN.build(model, dims, dec, seed=4, gin_eps=0.1)
    if pair == "dense_coo":
        ref.default_pair = (ag.KernelKind.DENSE_BLOCK, ag.KernelKind.COO_ATOMIC)
    net = D.DistGNN.build(model, dims, dec, rank=0, world=1, seed=4, gin_eps=0.1, pair=pair)
    V = rg.num_vertices
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn((V, dims[0]), device="cuda", generator=g)
    labels, mask = _labels_mask(V, dims[-1])
    n = int(mask.sum())
    loss_r, grads_r = ref.train_step(x, labels, mask, n, lr=0.0)
    loss_d, grads_d = net.train_step(net.input_ext(x), labels, mask, n, lr=0.0)
    tol = 1e-6 if pair == "csr" else 1e-5
    assert abs(loss_r.item() - loss_d.item()) <= tol * max(1.0, abs(loss_r.item()))
    for a, b in zip(grads_r, grads_d):
        assert rel_error(to_np(b), to_np(a)) < tol


@pytest.mark.parametrize("world,pair", [(2, "csr"), (4, "csr"), (2, "dense_coo")])
@pytest.mark.parametrize("model", ["gcn", "gin"])
def test_virtual_ranks_distgnn_step(world, pair, model):
    """G ranks as threads on one GPU (in-process all-to-all / all-reduce):
    the row-partitioned, reassociated step with the halo exchange and the
    overlapped backward equals the 1-GPU GNN step -- loss and every dW
    within 1e-5 -- and the per-peer halo never exceeds the padded all-gather."""
    import threading
    rg, dec = _setup(model, V=6000, E=80000)
    dims = [36, 64, 20, 7]  # a widening, then two narrowing (gemm-first) layers
    ref = ag.GNN.build(model, dims, dec, seed=2, gin_eps=0.2)
    V = rg.num_vertices
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn((V, dims[0]), device="cuda", generator=g)
    labels, mask = _labels_mask(V, dims[-1], seed=6)
    n = int(mask.sum())
    loss_r, grads_r = ref.train_step(x, labels, mask, n, lr=0.0)
    torch.cuda.synchronize()
    nets = [D.DistGNN.build(model, dims, dec, rank=r, world=world, seed=2, gin_eps=0.2,
                            subject_t=ref.subject_t, pair=pair) for r in range(world)]
    shared, barrier = {}, threading.Barrier(world)
    results, errors = {}, []
    for r, net in enumerate(nets):
        net.comm = ThreadComm(r, world, shared, barrier)
        st = net.fwd.plan.stats()
        assert st["halo_rows"] <= st["allgather_rows"]

    def run(r):
        try:
            net = nets[r]
            r0, r1 = net.bounds[r], net.bounds[r + 1]
            loss, grads = net.train_step(net.input_ext(x[r0:r1].contiguous()),
                                         labels[r0:r1].contiguous(), mask[r0:r1].contiguous(),
                                         n, lr=0.0)
            torch.cuda.synchronize()
            results[r] = (loss.clone(), [gr.clone() for gr in grads])
        except Exception as e:  # noqa: BLE001
            errors.append(e)
            barrier.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for r in range(world):
        loss_d, grads_d = results[r]
        assert abs(loss_r.item() - loss_d.item()) <= 1e-5 * max(1.0, abs(loss_r.item()))
        for a, b in zip(grads_r, grads_d):
            assert rel_error(to_np(b), to_np(a)) < 1e-5
