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
    for j, S in enumerate(plan.sets):
        base = plan.halo_base + j * plan.max_send
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
    for rank in range(world):
        op = D.LocalOperator.build(csr.row_ptr, csr.col_idx, csr.kernel_val, bounds, rank, B,
                                   mid=mid, role_col=rcol, role_val=rval,
                                   deg=dec.full_in_degree)
        x_ext = op.plan.new_ext(F, "cuda")
        _fill_halo(op.plan, x_ext, x)
        r0, r1 = bounds[rank], bounds[rank + 1]
        got = net.aggregate(op, x_ext, relu_src=h[r0:r1].contiguous())
        assert torch.equal(got, want[r0:r1]), (world, rank)


@pytest.mark.parametrize("model", ["gcn", "gin"])
def test_world1_distgnn_equals_gnn(model, monkeypatch):
    rg, dec = _setup(model, V=3000, E=30000)
    dims = [32, 24, 16, 5]
    ref = ag.GNN.build(model, dims, dec, seed=4, gin_eps=0.1)
    ref.reassociate = False  # DistGNN keeps the reference's aggregate-first order
    net = D.DistGNN.build(model, dims, dec, rank=0, world=1, seed=4, gin_eps=0.1)
    V = rg.num_vertices
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn((V, dims[0]), device="cuda", generator=g)
    rng = np.random.default_rng(5)
    labels = torch.from_numpy(rng.integers(0, dims[-1], V).astype(np.int32)).cuda()
    mask = torch.from_numpy(rng.random(V) < 0.5).cuda()
    n = int(mask.sum())
    loss_r, grads_r = ref.train_step(x, labels, mask, n, lr=0.0)
    loss_d, grads_d = net.train_step(net.input_ext(x), labels, mask, n, lr=0.0)
    assert abs(loss_r.item() - loss_d.item()) <= 1e-6 * max(1.0, abs(loss_r.item()))
    for a, b in zip(grads_r, grads_d):
        assert rel_error(to_np(b), to_np(a)) < 1e-6
