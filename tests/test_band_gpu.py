"""The band kernel (ag_band_spmm): the order-free (dense_block, coo_atomic)
selector pair with per-block topology records staged in shared memory.
Checked against the numpy restatement of the reference pair (kernels.py:
228-250 dense intra, :192-225 coo inter, :253-276 combine) at 1e-5, and
against the slab kernel running the same pair (AG_BAND=0; the band kernel is
opt-in, AG_BAND=1), on graphs that hit
each of its paths: ring sources, staged far rows, far-ring overflow to global
memory (rows flagged kRowGlobal), blocks past the staging capacity (pairs read
from the global record), windows wider than the band ring, partial last blocks
and column tiles, several row ranges per CTA, and every epilogue."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2305_17408_b200 as ag  # noqa: E402
from paper_2305_17408_b200 import _lib  # noqa: E402
from paper_2305_17408_b200 import kernels as K  # noqa: E402
from paper_2305_17408_b200.decompose import full_graph  # noqa: E402
from oracle import ref_numpy as R  # noqa: E402
from conftest import rel_error, to_np  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _band_on(monkeypatch):
    monkeypatch.setenv("AG_BAND", "1")
    monkeypatch.setenv("AG_GATHER", "0")  # these small graphs would take the gather pair
DENSE_COO = dict(kernel_intra=ag.KernelKind.DENSE_BLOCK, kernel_inter=ag.KernelKind.COO_ATOMIC)


def _community(V, E, window, p_global, model="gcn", skew=1, seed=0):
    from paper_2305_17408_b200 import synth
    g, comm = synth.community_graph(V, E, block_gen=16, p_intra=0.4, p_global=p_global,
                                    window=window, skew=skew, seed=seed)
    if model == "gcn":
        g = ag.gcn_normalize(g)
    rg = ag.apply_reorder(g, ag.reorder.partition_from_ids(comm, 16))
    return rg, ag.decompose(rg, 16)


def _oracle_pair(rg, x):
    V = rg.num_vertices
    d, s = to_np(rg.dst), to_np(rg.src)
    w = None if rg.weights is None else to_np(rg.weights)
    intra, inter, deg = R.decompose(V, d, s, w, 16)
    return R.aggregate_decomposed_csr(V, intra, inter, deg, x, "sum")


def _slab(monkeypatch, fn):
    monkeypatch.setenv("AG_BAND", "0")
    try:
        return fn()
    finally:
        monkeypatch.setenv("AG_BAND", "1")


def _band_used(dec):
    return K.to_csr(full_graph(dec))._band is not None


@pytest.mark.parametrize("F", [36, 48, 64, 100, 256])
def test_band_matches_oracle_and_slab(F, monkeypatch):
    rg, dec = _community(6001, 90000, window=6, p_global=0.05)
    x = np.random.default_rng(F).standard_normal((rg.num_vertices, F)).astype(np.float32)
    got = to_np(ag.aggregate_decomposed(dec, x, ag.AggregateOp.SUM, **DENSE_COO))
    assert _band_used(dec)
    assert rel_error(got, _oracle_pair(rg, x)) < 1e-5
    slab = _slab(monkeypatch, lambda: to_np(ag.aggregate_decomposed(dec, x, ag.AggregateOp.SUM,
                                                                     **DENSE_COO)))
    assert rel_error(got, slab) < 1e-5


@pytest.mark.parametrize("window,p_global", [(24, 0.05), (6, 0.45)])
def test_band_wide_window_and_far_overflow(window, p_global):
    """A window wider than the band ring (more far sources) and so many far
    sources that the 20-row far ring overflows to global loads."""
    rg, dec = _community(20000, 300000, window=window, p_global=p_global, seed=2)
    csr = K.to_csr(full_graph(dec))
    rec, off, far_cnt, far_src, win = csr.band_layout()
    idx = off[:-1].long()[:, None] * 4 + torch.arange(16, device=off.device)
    words = rec[idx].cpu().numpy().view(np.uint32)  # the 16 row words of every block
    assert ((words >> 20) & 0xFF).any(), "no row has far (global) sources"
    assert win <= int(_lib.load().ag_band_max_window())
    x = np.random.default_rng(1).standard_normal((rg.num_vertices, 128)).astype(np.float32)
    got = to_np(ag.aggregate_decomposed(dec, x, ag.AggregateOp.SUM, **DENSE_COO))
    assert rel_error(got, _oracle_pair(rg, x)) < 1e-5


def test_band_unstaged_blocks_and_hubs():
    """Hub rows: blocks with more inter pairs than the staging capacity read
    their pairs from the global record."""
    rg, dec = _community(30000, 600000, window=6, p_global=0.05, skew=2, seed=3)
    csr = K.to_csr(full_graph(dec))
    rec, off, _, _, _ = csr.band_layout()
    sizes = (off[1:] - off[:-1]).cpu().numpy() * 16
    cap = int(_lib.load().ag_band_capacity())
    assert (sizes > 64 + 8 * cap).any(), "no block exceeded the staging capacity"
    x = np.random.default_rng(2).standard_normal((rg.num_vertices, 64)).astype(np.float32)
    got = to_np(ag.aggregate_decomposed(dec, x, ag.AggregateOp.SUM, **DENSE_COO))
    assert rel_error(got, _oracle_pair(rg, x)) < 1e-4  # hub rows of ~2000 terms in fp32


def test_band_records_decode_to_role_layout():
    """Every record lists exactly the row's inter edges of the B = 16 role
    layout, in order, with their weights."""
    rg, dec = _community(3001, 40000, window=20, p_global=0.1, seed=5)
    csr = K.to_csr(full_graph(dec))
    mid, col, val = (to_np(t) for t in csr.role_layout(16))
    row_ptr = to_np(csr.row_ptr)
    rec, off, far_cnt, far_src, win = csr.band_layout()
    rec, off = to_np(rec), to_np(off)
    far_cnt, far_src = to_np(far_cnt), to_np(far_src)
    cap_far = int(_lib.load().ag_slab_far_capacity())
    V = rg.num_vertices
    for b in range((V + 15) // 16):
        words = rec[off[b] * 4: off[b] * 4 + 16].view(np.uint32)
        pairs = rec[off[b] * 4 + 16: off[b + 1] * 4].reshape(-1, 2)
        start = 0
        far_seen = []
        for i in range(16):
            r = 16 * b + i
            end = int(words[i] & 0xFFFFF)
            nfar = int((words[i] >> 20) & 0xFF)
            if r >= V:
                assert end == start
                continue
            cols = col[mid[r]:row_ptr[r + 1]]
            vals = val[mid[r]:row_ptr[r + 1]]
            near = np.abs(cols // 16 - b) <= win
            assert end - start == cols.size and nfar == int((~near).sum())
            order = np.concatenate([np.flatnonzero(~near), np.flatnonzero(near)])
            for (code, wb), c, v, nr in zip(pairs[start:end], cols[order], vals[order], near[order]):
                assert np.int32(wb).view(np.float32) == v
                if nr:
                    assert code == (c // 16) % 42 * 16 + c % 16
                else:
                    assert ~code == c
                    if c not in far_seen:
                        far_seen.append(c)
            start = end
        k = min(len(far_seen), cap_far)
        assert far_cnt[b] == k and list(far_src[b * cap_far: b * cap_far + k]) == far_seen[:k]


def test_band_epilogues_and_relu_bits(monkeypatch):
    """GIN (1 + eps) x term, the ReLU-backward mask (staged bits), and a
    forward ReLU writing relu bits -- bitwise equal bits to the slab kernel."""
    rg, dec = _community(8003, 100000, window=5, p_global=0.05, model="gin")
    rng = np.random.default_rng(4)
    for F in (48, 256):
        x = torch.from_numpy(rng.standard_normal((rg.num_vertices, F)).astype(np.float32)).cuda()
        h = torch.from_numpy(rng.standard_normal((rg.num_vertices, F)).astype(np.float32)).cuda()
        y = torch.empty_like(x)
        K.run_fused_pair(dec, x, y, ag.AggregateOp.SUM, 1.25, relu_src=h, **DENSE_COO)
        want = np.float32(1.25) * to_np(x) + _oracle_pair(rg, to_np(x))
        want = np.where(to_np(h) > 0, want, np.float32(0.0))
        assert rel_error(to_np(y), want) < 1e-5
        bits = K.relu_bits_empty(rg.num_vertices, F, x.device)
        y2 = torch.empty_like(x)
        K.run_fused_pair(dec, x, y2, ag.AggregateOp.SUM, relu=True, relu_out=bits, **DENSE_COO)
        ref = np.maximum(_oracle_pair(rg, to_np(x)), 0)
        assert rel_error(to_np(y2), ref) < 1e-5
        assert torch.equal(bits, K.relu_bits(y2))


def test_band_large_graph_repeatable():
    """Many blocks per CTA (the producers, dense warps and consumers drift
    apart): three launches agree with the bitwise CSR pair within 1e-5."""
    rg, dec = _community(300000, 4000000, window=12, p_global=0.05)
    x = torch.randn((rg.num_vertices, 100), device="cuda")
    want = torch.empty_like(x)
    K.run_fused_pair(dec, x, want, ag.AggregateOp.SUM)
    for _ in range(3):
        y = torch.empty_like(x)
        K.run_fused_pair(dec, x, y, ag.AggregateOp.SUM, **DENSE_COO)
        assert rel_error(to_np(y), to_np(want)) < 1e-5
