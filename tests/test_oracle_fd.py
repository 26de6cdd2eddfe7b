"""CPU: validate the composed training oracle (oracle/ref_numpy.py:gnn_step)
by central finite differences, the pattern of the reference's gradient
criterion (test_acceptance.py:239-260: 1/2 ||A X||^2 against backward_sum).

The composition (loss, layer backward, ReLU masks, the GIN (1+eps) term) is
builder-defined; every GPU training-step test compares with
gnn_step, so gnn_step itself is checked here against the derivative of its
own forward.  The check runs in fp64 (R.F32 patched to float64) so the
central difference is accurate to ~1e-9 and the tolerance can be tight.
"""
import numpy as np
import pytest

from conftest import random_graph_arrays
from oracle import ref_numpy as R


def _dense_adj(V, d, s, w):
    a = np.zeros((V, V), np.float64)
    np.add.at(a, (d, s), 1.0 if w is None else w.astype(np.float64))
    return a


def _loss_only(model, a, x, weights, labels, mask, eps):
    """Forward + loss of gnn_step's composition, fp64."""
    sc = 1.0 + eps
    h = x
    L = len(weights)
    for l in range(L):
        agg = a @ h
        if model == "gin":
            agg = sc * h + agg
        h = agg @ weights[l]
        if l < L - 1:
            h = np.maximum(h, 0.0)
    z = h - h.max(axis=1, keepdims=True)
    lp = z - np.log(np.exp(z).sum(axis=1, keepdims=True))
    rows = np.flatnonzero(mask)
    return float(-lp[rows, labels[rows]].sum() / rows.size)


@pytest.mark.parametrize("model,dims,eps", [("gcn", [6, 5, 4, 3], 0.0),
                                            ("gin", [5, 4, 4, 3], 0.25),
                                            ("gcn", [4, 7, 3], 0.0)])
def test_gnn_step_matches_finite_differences(monkeypatch, model, dims, eps):
    monkeypatch.setattr(R, "F32", np.float64)
    rng = np.random.default_rng(7)
    V, d, s, w = random_graph_arrays(rng, num_vertices=24, density=0.15, weighted=True)
    if model == "gcn":
        d, s, w = R.gcn_normalize(V, *R.canonical(V, d, s)[:2])
    a = _dense_adj(V, d, s, w)
    x = rng.standard_normal((V, dims[0]))
    weights = [rng.uniform(-0.6, 0.6, (dims[i], dims[i + 1])) for i in range(len(dims) - 1)]
    labels = rng.integers(0, dims[-1], V)
    mask = rng.random(V) < 0.6
    loss, grads, _ = R.gnn_step(model, lambda h: a @ h, lambda g: a.T @ g, x, weights, labels,
                                mask, gin_eps=eps)
    assert abs(loss - _loss_only(model, a, x, weights, labels, mask, eps)) < 1e-12
    h = 1e-6
    checked = 0
    for l, wl in enumerate(weights):
        for _ in range(6):
            i, j = int(rng.integers(wl.shape[0])), int(rng.integers(wl.shape[1]))
            wp = [q.copy() for q in weights]
            wm = [q.copy() for q in weights]
            wp[l][i, j] += h
            wm[l][i, j] -= h
            fd = (_loss_only(model, a, x, wp, labels, mask, eps) -
                  _loss_only(model, a, x, wm, labels, mask, eps)) / (2 * h)
            # the reference's FD criterion is abs < 1e-4; fp64 allows far tighter
            assert abs(fd - grads[l][i, j]) < 1e-7, (l, i, j, fd, grads[l][i, j])
            checked += 1
    assert checked == 6 * len(weights)


def test_layer_backward_formulas_match_finite_differences():
    """The single-layer backward the GPU gcn/gin_layer_backward implement:
    d_w = agg^T d_out, d_x = A^T (d_out W^T) [+ (1+eps) d_out W^T], checked on
    L = <d_out, layer(x)> by central differences in x and W."""
    rng = np.random.default_rng(3)
    V, d, s, w = random_graph_arrays(rng, num_vertices=20, density=0.2, weighted=True)
    a = _dense_adj(V, d, s, w)
    x = rng.standard_normal((V, 5))
    wt = rng.uniform(-0.5, 0.5, (5, 3))
    d_out = rng.standard_normal((V, 3))
    for eps in (None, 0.5):
        sc = 0.0 if eps is None else 1.0 + eps

        def f(xx, ww):
            return float(((sc * xx + a @ xx) @ ww * d_out).sum())

        agg = sc * x + a @ x
        d_w = agg.T @ d_out
        d_h = d_out @ wt.T
        d_x = a.T @ d_h + sc * d_h
        h = 1e-6
        for _ in range(8):
            i, j = int(rng.integers(V)), int(rng.integers(5))
            xp, xm = x.copy(), x.copy()
            xp[i, j] += h
            xm[i, j] -= h
            assert abs((f(xp, wt) - f(xm, wt)) / (2 * h) - d_x[i, j]) < 1e-7
            k, c = int(rng.integers(5)), int(rng.integers(3))
            wp, wm = wt.copy(), wt.copy()
            wp[k, c] += h
            wm[k, c] -= h
            assert abs((f(x, wp) - f(x, wm)) / (2 * h) - d_w[k, c]) < 1e-7
