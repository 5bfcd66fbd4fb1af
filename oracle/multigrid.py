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
                 nu_pre=1, nu_post=1, weight_mode="pou", bc="dirichlet"):
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


def vcycle(H, r, l=None):
    """z = B r with zero initial guess (PAPER.md:361-366 V-cycle preconditioner)."""
    if l is None:
        l = len(H.levels) - 1
    L = H.levels[l]
    prob = L.prob
    if l == 0:
        return H.coarse(r)
    u = np.zeros_like(r)
    for _ in range(H.nu_pre):
        u = smoother.wr_sweep(prob, prob.A, u, r, L.factors, H.omega_mg, L.w)
    res = r - prob.A @ u
    rc = transfer.restrict(H.P0[l], res, prob.NT)
    ec = vcycle(H, rc, l - 1)
    u = u + transfer.prolong(H.P0[l], ec, prob.NT)
    for _ in range(H.nu_post):
        u = smoother.wr_sweep(prob, prob.A, u, r, L.factors, H.omega_mg, L.w)
    return u
