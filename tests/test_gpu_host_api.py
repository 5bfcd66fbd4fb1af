"""wrmg_fgmres_host (the serving form of H13 on host buffers; the bench's end-to-end
leg): every right-hand side gives the device solve's iteration count and iterate."""
import numpy as np
import pytest
import torch

import wrmg_inputs as wi

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pinned", [True, False])
def test_fgmres_host_matches_device_solves(pinned):
    import paper_2407_13997_b200 as w
    n, k, q, N = 16, 3, 1, 12
    c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / N)
    lay = c.layout
    bs, xs, ref = [], [], []
    for seed in range(3):
        f = c.empty()
        c.fill_uniform(f, 0, seed)
        b = c.empty()
        c.rhs(f, b)
        x = c.empty()
        its, rel, st = c.fgmres(b, x, restart=30, maxit=100, rtol=1e-9)
        assert st == "WRMG_OK"
        ref.append((its, x.cpu().numpy()))
        hb = b.cpu()
        bs.append(hb.pin_memory() if pinned else hb)
        hx = torch.empty_like(hb)
        xs.append(hx.pin_memory() if pinned else hx)
    its_h, rel_h, st_h = c.fgmres_host(bs, xs, restart=30, maxit=100, rtol=1e-9)
    assert st_h == "WRMG_OK"
    for i, (its, xr) in enumerate(ref):
        assert its_h[i] == its
        assert rel_h[i] <= 1e-9 * 1.001
        xg = xs[i].numpy()
        assert np.linalg.norm(xg - xr) <= 1e-12 * np.linalg.norm(xr)
    assert lay["ndof"] == xs[0].numel()
    c.close()


def test_stationary_equals_explicit_cycles():
    """wrmg_stationary (the C5 protocol's u <- u + V(b - A u), all in the library) equals
    the same cycles composed from wrmg_residual / wrmg_vcycle."""
    import paper_2407_13997_b200 as w
    n, k, q, N = 16, 2, 1, 10
    c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / N)
    f = c.empty()
    c.fill_uniform(f, 0, 0)
    b = c.empty()
    c.rhs(f, b)
    u1 = c.zeros()
    c.stationary(b, u1, 3)
    u2, r, z = c.zeros(), c.empty(), c.empty()
    for _ in range(3):
        c.residual(u2, b, r)
        c.vcycle(r, z)
        u2 += z
    torch.cuda.synchronize()
    a1, a2 = u1.cpu().numpy(), u2.cpu().numpy()
    assert np.linalg.norm(a1 - a2) <= 1e-12 * np.linalg.norm(a2)
    c.close()
