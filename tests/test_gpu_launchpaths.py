"""GPU parity on the launch configurations the small parity cases never reach
(ADVICE r01): full vectors against the oracle.

* the DMMA Kronecker sweep ``k_sweep_kron_mma<MP>`` runs on DG1 levels with at
  least 1000 patches: MP = 7 (P2, 32x32, 1087 patches), MP = 1 (P1, 48x48, 2209
  patches) and MP = 19 (P3, 40x40, 1681 patches), each with N crossing its
  16-slab chunks (N = 40 / 20) -- three sweeps, one V(1,1), and FGMRES (identical
  iteration counts; P1 x DG1 with V(1,1) does not converge, so its first 6
  iterations are compared);
* the multi-patch CTA plan of ``k_sweep_kron`` (PP = 8 patches per CTA) runs on
  levels with one 32-slab chunk and at least 2 x 148 CTAs: q = 0 and q = 2 on a
  50x50 mesh (2401 / 2601 patches), every entry of three sweeps.
"""
import numpy as np
import pytest

import wrmg_inputs as wi
from test_gpu_parity import TOL, _dev, _host, assert_parity

pytestmark = pytest.mark.gpu


def _setup(n, k, q, N, nc):
    import paper_2407_13997_b200 as w
    from oracle import multigrid
    H = multigrid.Hierarchy(n, n, 1.0 / n, k, q, N, 1.0 / N, n_coarse=nc)
    c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / N, ncoarse=nc)
    assert c.layout["nlevels"] == len(H.levels)
    return H, c


@pytest.mark.parametrize("n,k,N,nc,mp", [(32, 2, 40, 4, 7), (48, 1, 40, 4, 1), (40, 3, 20, 5, 19)])
def test_dmma_sweep_vcycle_fgmres(n, k, N, nc, mp):
    from oracle import krylov, multigrid, smoother
    q = 1
    H, c = _setup(n, k, q, N, nc)
    p = H.fine
    L = H.levels[-1]
    assert c.layout["npatch"] >= 1000 and c.layout["mp_max"] == mp  # the DMMA sweep's launch condition
    b = p.rhs(wi.spacetime_field(p.nnode, N, q, 0))
    db = _dev(b)
    u0 = wi.spacetime_field(p.nnode, N, q, 2) * ~p.con_st
    u_ref, u = u0.copy(), _dev(u0)
    for s, om in enumerate((1.0, 0.8, 1.0)):
        u_ref = smoother.wr_sweep(p, p.A, u_ref, b, L.factors, om, L.w)
        c.smooth(u, db, 1, om)
        assert_parity(_host(u), u_ref, what=f"sweep {s}")
    z = c.empty()
    c.vcycle(db, z)
    assert_parity(_host(z), multigrid.vcycle(H, b), what="V(1,1)")
    maxit = 200 if k > 1 else 6
    x_ref, its_ref, hist, st = krylov.fgmres(lambda v: p.A @ v, lambda r: multigrid.vcycle(H, r), b,
                                             restart=30, maxit=maxit, rtol=1e-8)
    x = c.empty()
    its, rel, status = c.fgmres(db, x, restart=30, maxit=maxit, rtol=1e-8)
    assert its == its_ref, (its, its_ref)
    if k > 1:
        assert status == "WRMG_OK" and st == "converged"
    assert_parity(_host(x), x_ref, tol=1e-9, what="fgmres iterate")
    c.close()


@pytest.mark.parametrize("k,q", [(1, 0), (2, 2)])
def test_multi_patch_cta_sweep(k, q):
    from oracle import patches, smoother
    from oracle import heat
    import paper_2407_13997_b200 as w
    n, N = 50, 4
    p = heat.unit_square_problem(n, k, q, N, 1.0 / N)
    c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / N)
    P, _ = patches.vertex_star_patches(p.mesh, k, p.constrained)
    assert len(P) // 8 >= 2 * 148  # PP = 8 (one 32-slab chunk) is kept: >= 2 CTAs per SM
    fac = smoother.PatchFactors(p, p.A, P)
    wts = smoother.weights(P, p.nnode)
    b = p.rhs(wi.spacetime_field(p.nnode, N, q, 0))
    u0 = wi.spacetime_field(p.nnode, N, q, 5) * ~p.con_st
    u_ref, u = u0.copy(), _dev(u0)
    for s, om in enumerate((0.6, 1.0, 1.0)):
        u_ref = smoother.wr_sweep(p, p.A, u_ref, b, fac, om, wts)
        c.smooth(u, _dev(b), 1, om)
        assert_parity(_host(u), u_ref, tol=TOL, what=f"sweep {s}")
    c.close()
