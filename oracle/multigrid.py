"""Space-time semi-coarsened geometric multigrid.

Hierarchy {t_n} (x) T_H, ..., {t_n} (x) T_h: the spatial mesh is coarsened by
two, the temporal mesh is the same on every level.  Coarse
operators are rediscretised (R13); the coarsest level has n_c cells
in the shorter direction (R14, default 4) and is solved exactly by
block forward substitution in time with a dense LU of each slab block
(R10).  The V-cycle is V(nu_pre, nu_post) with the weighted additive
waveform smoother (R15: V(1,1), omega_mg); used as a preconditioner it
starts from a zero guess.
"""
import numpy as np
import scipy.linalg as sla

from . import heat, smoother, transfer
from . import patches as patchmod
from .mesh import Mesh


class Level:
    def __init__(self, prob, weight_mode):
        self.prob = prob
        self.patches, self.patch_vertices = patchmod.vertex_star_patches(prob.mesh, prob.k, prob.constrained)
        self.w = smoother.weights(self.patches, prob.nnode, weight_mode)
        self.factors = smoother.PatchFactors(prob, prob.A, self.patches)


class Hierarchy:
    def __init__(self, nx, ny, h, k, q, N, dt, kappa=1.0, n_coarse=4, omega_mg=1.0,
                 nu_pre=1, nu_post=1, weight_mode="pou", bc="dirichlet", smoother_kind="damped", cheb_steps=50,
                 cheb_seed=7):
        meshes = [Mesh(nx, ny, h)]
        while min(meshes[-1].nx, meshes[-1].ny) > n_coarse:
            m = meshes[-1]
            assert m.nx % 2 == 0 and m.ny % 2 == 0
            meshes.append(Mesh(m.nx // 2, m.ny // 2, 2 * m.h))
        meshes = meshes[::-1]  # coarse -> fine
        self.levels = [Level(heat.HeatProblem(m, k, q, N, dt, kappa, bc=bc), weight_mode) for m in meshes]
        self.coarse = CoarseSolver(self.levels[0].prob)
        self.P0 = [None]
        for l in range(1, len(self.levels)):
            cp, fp = self.levels[l - 1].prob, self.levels[l].prob
            P = transfer.interpolation(cp.mesh, fp.mesh, k)
            self.P0.append(transfer.correction_interpolation(P, fp.constrained, cp.constrained))
        self.omega_mg, self.nu_pre, self.nu_post = omega_mg, nu_pre, nu_post
        self.smoother_kind = smoother_kind
        self.lam = [None] * len(self.levels)
        if smoother_kind == "chebyshev":
            for l in range(1, len(self.levels)):
                self.lam[l] = estimate_lambda(self.levels[l], cheb_steps, cheb_seed)

    @property
    def fine(self):
        return self.levels[-1].prob


class CoarseSolver:
    """Exact solve of A x = r: for n = 0..N-1, x_n = D_n^{-1} (r_n - L_n x_{n-1})
    with D_n the full slab block (all nodes, constrained identity rows included),
    factored once per slab with LAPACK dgetrf."""

    def __init__(self, prob):
        A = prob.A
        nodes = np.arange(prob.nnode)
        self.prob = prob
        self.I = [prob.slab_indices(nodes, n) for n in range(prob.N)]
        self.lu = [sla.lu_factor(A[I][:, I].toarray()) for I in self.I]
        self.L = [None] + [A[self.I[n]][:, self.I[n - 1]].toarray() for n in range(1, prob.N)]

    def __call__(self, r):
        x = np.zeros_like(r)
        for n, I_n in enumerate(self.I):
            rhs = r[I_n].copy()
            if n > 0:
                rhs -= self.L[n] @ x[self.I[n - 1]]
            x[I_n] = sla.lu_solve(self.lu[n], rhs)
        return x


def relaxation(L, r):
    """B r: one additive WR sweep from zero with unit damping."""
    p = L.prob
    return smoother.wr_sweep(p, p.A, np.zeros_like(r), r, L.factors, 1.0, L.w)


def estimate_lambda(L, steps=50, seed=7):
    """Largest eigenvalue estimate of the relaxation-preconditioned operator B A
    ("50 steps of relaxation-preconditioned GMRES").  Reading
    (DESIGN.md R-cheb): `steps` Arnoldi steps (classical Gram-Schmidt twice) on B A
    from the seeded vector U[-1,1) at the canonical ids (generator of R6, `seed`,
    constrained rows 0), and the estimate is the largest modulus among the Ritz
    values (eigenvalues of the square steps x steps Hessenberg)."""
    import wrmg_inputs as wi
    p = L.prob
    v = wi.uniform_pm1(np.arange(p.ndof, dtype=np.uint64), seed)
    v[np.repeat(p.constrained, p.NT)] = 0.0
    V = [v / np.linalg.norm(v)]
    Hm = np.zeros((steps + 1, steps))
    for j in range(steps):
        w = relaxation(L, p.A @ V[j])
        Vm = np.array(V)
        h = Vm @ w
        w = w - Vm.T @ h
        h2 = Vm @ w
        w = w - Vm.T @ h2
        Hm[:j + 1, j] = h + h2
        Hm[j + 1, j] = np.linalg.norm(w)
        V.append(w / Hm[j + 1, j])
    return float(np.abs(np.linalg.eigvals(Hm[:steps, :steps])).max())


def chebyshev(L, u, b, lam, nu):
    """nu steps of Chebyshev iteration for B A x = B b on the interval
    [0.25 lam, 1.05 lam], three-term recurrence:
        theta = (b+a)/2, delta = (b-a)/2, sigma = theta/delta, rho_0 = 1/sigma,
        d_0 = B r_0 / theta,  d_k = rho_k rho_{k-1} d_{k-1} + (2 rho_k / delta) B r_k,
        rho_k = 1 / (2 sigma - rho_{k-1}),  x_{k+1} = x_k + d_k."""
    A = L.prob.A
    lo, hi = 0.25 * lam, 1.05 * lam
    theta, delta = 0.5 * (hi + lo), 0.5 * (hi - lo)
    sigma = theta / delta
    rho = 1.0 / sigma
    d = relaxation(L, b - A @ u) / theta
    u = u + d
    for _ in range(1, nu):
        rn = 1.0 / (2.0 * sigma - rho)
        d = rn * rho * d + (2.0 * rn / delta) * relaxation(L, b - A @ u)
        rho = rn
        u = u + d
    return u


def vcycle(H, r, l=None):
    """z = B r with zero initial guess (PAPER.md:361-366 V-cycle preconditioner);
    smoothing is nu damped additive WR sweeps (R15) or, with smoother_kind =
    "chebyshev", nu Chebyshev-accelerated steps."""
    if l is None:
        l = len(H.levels) - 1
    L = H.levels[l]
    prob = L.prob
    if l == 0:
        return H.coarse(r)
    cheb = H.smoother_kind == "chebyshev"
    u = np.zeros_like(r)
    if cheb:
        u = chebyshev(L, u, r, H.lam[l], H.nu_pre)
    else:
        for _ in range(H.nu_pre):
            u = smoother.wr_sweep(prob, prob.A, u, r, L.factors, H.omega_mg, L.w)
    res = r - prob.A @ u
    rc = transfer.restrict(H.P0[l], res, prob.NT)
    ec = vcycle(H, rc, l - 1)
    u = u + transfer.prolong(H.P0[l], ec, prob.NT)
    if cheb:
        u = chebyshev(L, u, r, H.lam[l], H.nu_post)
    else:
        for _ in range(H.nu_post):
            u = smoother.wr_sweep(prob, prob.A, u, r, L.factors, H.omega_mg, L.w)
    return u
