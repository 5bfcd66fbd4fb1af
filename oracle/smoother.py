"""Waveform-relaxation additive patch smoother.

"vertex-star relaxation in the spatial domain, extended (in the usual style of
waveform relaxation) to couple all degrees of freedom in space-time that reside
in the spatial patch".  For patch p with space-time index set
I_p (its spatial DoFs over every slab):

    A_p = A[I_p, I_p]                       (R9: R_p A R_p^T)

is block lower-bidiagonal in time, with diagonal blocks D_{p,n} and
sub-diagonal blocks L_{p,n}.  One sweep (R11):

    r   = b - A u
    for each patch p, for n = 0..N-1 in order:
        x_{p,n} = D_{p,n}^{-1} (r[I_{p,n}] - L_{p,n} x_{p,n-1})    (dense LU per (p, n), R10)
    u  <- u + omega * sum_p R_p^T W_p x_p,   W_p = diag(1/mu_i)

The LU is scipy.linalg.lu_factor (LAPACK dgetrf, partial pivoting).  The
factorisation of every (p, n) block is computed once per operator
(``PatchFactors``) and reused by every sweep, as the method does (factor at
setup / linearisation, apply in every sweep).
"""
import numpy as np
import scipy.linalg as sla

from . import patches as patchmod


def patch_indices(prob, patch):
    """Space-time indices of a patch, slab-major: concat_n slab_indices(patch, n)."""
    return np.concatenate([prob.slab_indices(patch, n) for n in range(prob.N)])


class PatchFactors:
    """LU factors of D_{p,n} and dense L_{p,n} for every patch p and slab n."""

    def __init__(self, prob, A, patches):
        self.prob, self.patches = prob, patches
        self.I = []
        self.lu = []
        self.L = []
        for p in patches:
            I_p = patch_indices(prob, p)
            Ap = A[I_p][:, I_p].tocsr()
            m = p.size * (prob.q + 1)
            lus, Ls = [], []
            for n in range(prob.N):
                D = Ap[n * m:(n + 1) * m, n * m:(n + 1) * m].toarray()
                lus.append(sla.lu_factor(D))
                Ls.append(Ap[n * m:(n + 1) * m, (n - 1) * m:n * m].toarray() if n > 0 else None)
            self.I.append(I_p)
            self.lu.append(lus)
            self.L.append(Ls)

    def solve(self, pi, g):
        """Exact solve of A_p x = g by forward substitution over slabs."""
        m = self.patches[pi].size * (self.prob.q + 1)
        x = np.zeros_like(g)
        for n in range(self.prob.N):
            rhs = g[n * m:(n + 1) * m].copy()
            if n > 0:
                rhs -= self.L[pi][n] @ x[(n - 1) * m:n * m]
            x[n * m:(n + 1) * m] = sla.lu_solve(self.lu[pi][n], rhs)
        return x


def patch_blocks_kron(prob, patch):
    """D_{p,n} and L_{p,n} (same for every slab of the heat operator) from the
    Kronecker definition of A (heat.py) restricted to the patch's free rows and
    columns, without forming A: D = M_pp (x) (C+E0) + kappa K_pp (x) Mt,
    L = -M_pp (x) E1 (node-major, temporal node fastest, like slab_indices).
    Identical to A[I_p][:, I_p] for patches of free DoFs (R9); pinned by
    tests/test_oracle_solver.py::test_patch_blocks_kron_equal_restriction."""
    tm = prob.tm
    Mpp = prob.M[patch][:, patch].toarray()
    Kpp = prob.K[patch][:, patch].toarray()
    D = np.kron(Mpp, tm.C + tm.E0) + prob.kappa * np.kron(Kpp, tm.Mt)
    L = -np.kron(Mpp, tm.E1)
    return D, L


def patch_solve_kron(prob, patch, g):
    """Forward substitution over slabs with the Kronecker-built blocks
    (dense LAPACK LU per slab); g, x slab-major like patch_indices."""
    D, L = patch_blocks_kron(prob, patch)
    m = D.shape[0]
    x = np.zeros_like(g)
    for n in range(prob.N):
        rhs = g[n * m:(n + 1) * m].copy()
        if n > 0:
            rhs -= L @ x[(n - 1) * m:n * m]
        x[n * m:(n + 1) * m] = sla.lu_solve(sla.lu_factor(D), rhs)
    return x


def weights(patches, nnode, mode="pou"):
    if mode == "pou":
        mu = patchmod.multiplicity(patches, nnode)
        w = np.zeros(nnode)
        w[mu > 0] = 1.0 / mu[mu > 0]
        return w
    if mode == "none":
        return np.ones(nnode)
    raise ValueError(mode)


def wr_sweep(prob, A, u, b, factors, omega, w_node, order=None):
    """One additive waveform-relaxation sweep; returns the new iterate."""
    r = b - A @ u
    du = np.zeros_like(u)
    idx = range(len(factors.patches)) if order is None else order
    for pi in idx:
        p = factors.patches[pi]
        I_p = factors.I[pi]
        x = factors.solve(pi, r[I_p])
        wt = np.repeat(w_node[p], prob.q + 1)  # slab block: node-major, a fastest
        du[I_p] += np.tile(wt, prob.N) * x
    return u + omega * du
