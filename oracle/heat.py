"""Space-time heat operator of eq. heatfem, with the
diffusion coefficient kappa, forcing f and Dirichlet data of BASELINE.json's
configs (R3, R5, R6, R7).

Unknowns U in DG(q) x CG(k), stored waveform-major (R4):
    index(i, n, a) = (i * N + n) * (q + 1) + a,
i the canonical lattice node, n the slab, a the temporal node.

Applying the temporal matrices of dg.py to eq. heatfem with forcing term
int (f, psi) gives, slab by slab,
    [(C + E0) (x) M + Mt (x) kappa K] U_n  -  (E1 (x) M) U_{n-1}  =  (Mt (x) M) f_n,
i.e. the block lower-bidiagonal matrix
    A = M (x) Tm + kappa K (x) Tk,
    Tm = I_N (x) (C + E0) - S_N (x) E1     (S_N: ones on the sub-diagonal),
    Tk = I_N (x) Mt,
where (x) is the Kronecker product in the waveform-major ordering
(space outermost).  Dirichlet DoFs are identity rows (R5), imposed at every
temporal node; the initial condition enters the RHS of slab 0 (R7).
"""
import numpy as np
import scipy.sparse as sp

from . import dg, fem
from . import mesh as meshmod


class HeatProblem:
    def __init__(self, mesh, k, q, N, dt, kappa=1.0, bc="dirichlet", build_matrix=True):
        self.mesh, self.k, self.q, self.N, self.dt = mesh, int(k), int(q), int(N), float(dt)
        self.kappa = float(kappa)
        self.bc = bc
        self.tm = dg.TemporalMatrices(q, dt)
        self.M, self.K = fem.assemble(mesh, k)
        self.nnode = self.M.shape[0]
        self.NT = self.N * (self.q + 1)
        if bc == "dirichlet":
            self.constrained = meshmod.boundary_nodes(mesh, k)
        elif bc == "neumann":
            self.constrained = np.zeros(self.nnode, dtype=bool)
        else:
            raise ValueError(bc)
        self.free = ~self.constrained
        nq = self.q + 1
        I_N = sp.identity(self.N, format="csr")
        S_N = sp.diags([np.ones(self.N - 1)], [-1], shape=(self.N, self.N), format="csr")
        self.Tm = (sp.kron(I_N, sp.csr_matrix(self.tm.C + self.tm.E0))
                   - sp.kron(S_N, sp.csr_matrix(self.tm.E1))).tocsr()
        self.Tk = sp.kron(I_N, sp.csr_matrix(self.tm.Mt)).tocsr()
        self.con_st = np.repeat(self.constrained, self.NT)
        self.A = self.spacetime_operator() if build_matrix else None

    @property
    def ndof(self):
        return self.nnode * self.NT

    def index(self, i, n, a):
        return (np.asarray(i) * self.N + np.asarray(n)) * (self.q + 1) + np.asarray(a)

    def spacetime_operator(self):
        A0 = sp.kron(self.M, self.Tm, format="csr") + self.kappa * sp.kron(self.K, self.Tk, format="csr")
        keep = sp.diags((~self.con_st).astype(float))
        ident = sp.diags(self.con_st.astype(float))
        A = (keep @ A0 + ident).tocsr()
        A.eliminate_zeros()
        return A

    def rhs(self, fhat, u0=None, bc_value=0.0):
        """b = (M (x) I_N (x) Mt) fhat on free rows (R6); the slab-0 jump term
        phi_a(0) (M u0)_i for an initial state u0 (R7, eq. dgintime Y_0^- = y_0);
        constrained rows carry the boundary value."""
        f2 = np.asarray(fhat, dtype=float).reshape(self.nnode, self.N, self.q + 1)
        Mf = (self.M @ f2.reshape(self.nnode, -1)).reshape(self.nnode, self.N, self.q + 1)
        b = np.einsum("ab,inb->ina", self.tm.Mt, Mf)
        if u0 is not None:
            Mu0 = self.M @ np.asarray(u0, dtype=float)
            b[:, 0, :] += np.outer(Mu0, self.tm.phi0)
        b = b.reshape(-1)
        b[self.con_st] = bc_value
        return b

    def residual(self, u, b):
        """r = b - A u (constrained rows: r = b - u)."""
        return b - self.A @ u

    def residual_rows(self, rows, u, b):
        """Selected rows of b - A u, evaluated from the Kronecker definition of A
        without forming it (for full-size sampled parity)."""
        rows = np.asarray(rows, dtype=np.int64)
        u2 = np.asarray(u, dtype=float).reshape(self.nnode, self.NT)
        out = np.empty(rows.size)
        Tm = self.Tm.toarray() if self.NT <= 4096 else None
        Tk = self.Tk.toarray() if self.NT <= 4096 else None
        for r_i, row in enumerate(rows):
            i, t = divmod(int(row), self.NT)
            if self.constrained[i]:
                out[r_i] = b[row] - u2[i, t]
                continue
            mrow = self.M.getrow(i)
            krow = self.K.getrow(i)
            mu = mrow @ u2  # (1, NT)
            ku = krow @ u2
            out[r_i] = b[row] - (np.ravel(mu) @ Tm[t] + self.kappa * (np.ravel(ku) @ Tk[t]))
        return out

    def residual_node(self, i, u, b):
        """All N (q+1) values of b - A u at spatial node i (Kronecker definition,
        without forming A; for full-size sampled parity)."""
        u2 = np.asarray(u, dtype=float).reshape(self.nnode, self.NT)
        bi = np.asarray(b, dtype=float).reshape(self.nnode, self.NT)[i]
        if self.constrained[i]:
            return bi - u2[i]
        mu = np.ravel(self.M.getrow(i) @ u2)
        ku = np.ravel(self.K.getrow(i) @ u2)
        return bi - (self.Tm @ mu + self.kappa * (self.Tk @ ku))

    def slab_indices(self, nodes, n):
        """Space-time indices of spatial nodes `nodes` in slab n, ordered
        (node-major, temporal node fastest)."""
        nodes = np.asarray(nodes, dtype=np.int64)
        a = np.arange(self.q + 1)
        return (self.index(nodes[:, None], n, a[None, :])).ravel()


def unit_square_problem(n, k, q, N, dt, **kw):
    return HeatProblem(meshmod.unit_square(n), k, q, N, dt, **kw)
