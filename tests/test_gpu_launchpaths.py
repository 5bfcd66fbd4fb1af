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


def test_multi_patch_cta_sweep():
    """P1 x DG0 on 50x50 (2401 single-node patches, one 32-slab chunk): PP = 8 patches
    per CTA in k_sweep_kron, every entry of three sweeps."""
    from oracle import patches, smoother
    from oracle import heat
    import paper_2407_13997_b200 as w
    n, k, q, N = 50, 1, 0, 4
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


def _sampled_sweep_check(n, k, q, N, nodes_ij, omega=0.9):
    """One sweep from a random state on an n x n mesh; the update at the sampled
    nodes against omega * sum_{p ni i} x_p[i] / mu_i, x_p = the oracle's exact patch
    space-time solve (Kronecker-built blocks, per-slab LAPACK LU)."""
    from oracle import heat, smoother
    from oracle import patches as pm
    import paper_2407_13997_b200 as w
    p = heat.unit_square_problem(n, k, q, N, 1.0 / N, build_matrix=False)
    c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / N)
    P, _ = pm.vertex_star_patches(p.mesh, k, p.constrained)
    b = wi.spacetime_field(p.nnode, N, q, seed=3)
    u0 = wi.spacetime_field(p.nnode, N, q, seed=4) * np.repeat(p.free, p.NT)
    ug = _dev(u0)
    c.smooth(ug, _dev(b), 1, omega)
    du = (_host(ug) - u0).reshape(p.nnode, -1)
    mu = pm.multiplicity(P, p.nnode)
    L = k * n + 1
    nq = q + 1
    rn = {}

    def rnode(j):
        if j not in rn:
            rn[j] = p.residual_node(j, u0, b).reshape(N, nq)
        return rn[j]

    worst = 0.0
    for I, J in nodes_ij:
        i = J * L + I
        if not p.free[i]:
            continue
        acc = np.zeros(p.NT)
        for pt in P:
            if i not in pt:
                continue
            g = np.concatenate([np.stack([rnode(j)[s] for j in pt]).ravel() for s in range(N)])
            x = smoother.patch_solve_kron(p, pt, g).reshape(N, pt.size, nq)
            acc += omega * x[:, list(pt).index(i), :].ravel() / mu[i]
        worst = max(worst, np.max(np.abs(du[i] - acc)) / np.max(np.abs(acc)))
    c.close()
    return worst


@pytest.mark.parametrize("n,k,q,N", [(40, 3, 0, 37), (40, 3, 2, 6), (40, 3, 1, 20), (36, 2, 0, 33),
                                     (36, 2, 2, 4), (36, 2, 3, 5), (48, 2, 1, 3),
                                     # chunk-parallel form (k_sweep_sym_cp): ragged groups, two groups
                                     (36, 3, 1, 70), (32, 2, 1, 150)])
def test_symmetric_sweep_sampled(n, k, q, N):
    """Levels with >= 1000 patches run the interior class through the symmetry-reduced
    sweep (kernels_sweep_sym.cu) and the boundary classes through kernels_kron.cu;
    sampled nodes cover the vertex, edge and cell-interior types of both, the corners
    and the lattice edges.  With N > 32 slabs and fewer than 8 four-patch CTAs per SM
    the chunk-parallel form runs (four warps = four 32-slab chunks of one patch)."""
    L = k * n + 1
    m = L // 2
    nodes = [(1, 1), (2, 1), (1, 2), (k, k), (k + 1, k), (2 * k, 1), (m, m), (m + 1, m), (m, m + 1),
             (m + 1, m + 2), (m + 2, m + 2), (L - 2, L - 2), (L - 2, m), (m, 1), (3 * k + 1, 2 * k + 2)]
    assert _sampled_sweep_check(n, k, q, N, nodes) <= 1e-10


@pytest.mark.parametrize("side", ["1", "0"])
def test_side_stream_boundary_sweep(monkeypatch, side):
    """WRMG_SWEEP_SIDE=1: the boundary classes' Kronecker sweep runs on a side stream
    concurrently with the symmetric class (opt-in); =0, the default, serialises them.  Both: full vectors of three
    sweeps, one V(1,1) and the FGMRES count against the oracle (P3 x DG1, 40 x 40)."""
    monkeypatch.setenv("WRMG_SWEEP_SIDE", side)
    test_dmma_sweep_vcycle_fgmres(40, 3, 20, 5, 19)
