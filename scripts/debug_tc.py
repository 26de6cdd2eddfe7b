"""Layout diagnostics for the tcgen05 GEMM (development aid, runs on the GPU box)."""
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2305_17408_b200 import kernels as K  # noqa: E402
import paper_2305_17408_b200 as ag  # noqa: E402


def show(name, got, ref):
    got, ref = got.double().cpu().numpy(), ref.double().cpu().numpy()
    err = np.abs(got - ref).max()
    print(f"{name}: max err {err:.3e}  got[:2,:6]={np.round(got[:2, :6], 2).tolist()} "
          f"ref[:2,:6]={np.round(ref[:2, :6], 2).tolist()}", flush=True)
    if err > 1e-3:
        bad = np.argwhere(np.abs(got - ref) > 1e-3)
        print("   first bad", bad[:6].tolist(), "count", len(bad), "of", got.size)
        # which ref element does got[m,n] equal?
        for m, n in bad[:4]:
            hits = np.argwhere(np.abs(ref - got[m, n]) < 1e-4)
            print(f"   got[{m},{n}]={got[m, n]:.3f} equals ref at {hits[:4].tolist()}")


def main():
    torch.manual_seed(0)
    for M, Kd, N in ((128, 32, 32), (128, 64, 64), (256, 100, 256)):
        a = torch.randint(-3, 4, (M, Kd), device="cuda").float()
        eye = torch.eye(Kd, N, device="cuda")
        b = torch.randint(-3, 4, (Kd, N), device="cuda").float()
        for ta in (False, True):
            for tb in (False, True):
                A = a.t().contiguous() if ta else a
                B = b.t().contiguous() if tb else b
                got = K.gemm(A, B, trans_a=ta, trans_b=tb, engine="tc")
                show(f"M{M} K{Kd} N{N} ta={ta} tb={tb} AB", got, a @ b)
                E = eye.t().contiguous() if tb else eye
                got = K.gemm(A, E, trans_a=ta, trans_b=tb, engine="tc")
                show(f"M{M} K{Kd} N{N} ta={ta} tb={tb} A*I", got, a @ eye)
        torch.cuda.synchronize()
    # aggregation: new fused kernel vs the reference-order CSR kernel
    rng = np.random.default_rng(0)
    V, E = 3000, 40000
    keys = rng.choice(V * V, size=E, replace=False)
    g = ag.gcn_normalize(ag.Graph.from_edges(V, keys // V, keys % V))
    csr = K.to_csr(g)
    for F in (1, 4, 16, 64, 100, 256):
        x = torch.randn((V, F), device="cuda")
        y_old = torch.empty_like(x)
        y_new = torch.empty_like(x)
        K.launch_csr(csr, x, y_old, ag.AggregateOp.SUM)
        K.launch_fused(csr, x, y_new, ag.AggregateOp.SUM)
        diff = (y_old != y_new).any(dim=1).nonzero().flatten()
        print(f"agg F={F}: rows differing {diff.numel()} / {V}", flush=True)
        if diff.numel():
            r = int(diff[0])
            rp = csr.row_ptr.cpu().numpy()
            print("   row", r, "deg", rp[r + 1] - rp[r], "old", y_old[r, :4].tolist(),
                  "new", y_new[r, :4].tolist())
            degs = (rp[1:] - rp[:-1])[diff.cpu().numpy()]
            print("   degrees of differing rows", np.bincount(degs)[:40].tolist())


if __name__ == "__main__":
    main()
