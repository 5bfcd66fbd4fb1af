"""Space-time Navier-Stokes (eq. nsfem) with Taylor-Hood
P_{k+1}-P_k in space and DG(q) in time, its Newton linearisation, Vanka+star
patches (Fig. patches right), the semi-coarsened V-cycle and
Newton-Krylov with Eisenstat-Walker forcing.

Unknowns: velocity components u_x, u_y on the P_{k+1} lattice (Lu nodes each) and
pressure on the P_k lattice (Lp nodes).  Combined spatial index ("sid"):
    u_x node i -> i,   u_y node i -> Lu + i,   p node j -> 2 Lu + j,
space-time index (sid * N + n) (q + 1) + a (R4, field order SPEC.md:150).

Per slab n, with test phi_a and trial phi_b (dg.py), the momentum rows read
    sum_b (C+E0)_ab M U_{n,b} - (E1 M U_{n-1})_a + Mt_ab K U_{n,b} + Mt_ab G P_{n,b}
      + R sum_{b,c} T_abc O(U_{n,c}) U_{n,b}
and the continuity rows sum_b Mt_ab G^T U_{n,b}, where
    M, K  = blockdiag(mass, stiffness) of P_{k+1} (both components),
    G[(d,i), j] = int chi_j d_d v_i   from +(Phi, div psi) (R17: the
                  velocity-pressure and pressure-velocity blocks are plain transposes),
    O(w)[(d,i),(d',j)] = delta_dd' int v_i (w . grad v_j)   (convection (U . grad) U),
    T_abc = dt int phi_a phi_b phi_c.
The jump acts on velocity only.  Newton Jacobian at W (R18):
the convection block of (a, b) is R sum_c T_abc N(W_{n,c}) with
    N(w) = O(w) + Q(w),  Q(w)[(d,i),(d',j)] = int v_i v_j d_d' w_d.
Dirichlet velocity DoFs are identity rows with the boundary value (R5); the
pressure is determined up to one constant per (slab, temporal node) and is
mean-projected (R19).
"""
import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from . import dg, fem, smoother, transfer
from . import mesh as meshmod
from .mesh import Mesh


def _assemble_th(mesh, ku, kp):
    """Global velocity mass/stiffness (scalar, Lu x Lu), divergence couplings
    G_d (Lu x Lp), and the cell data needed for convection."""
    vd = fem.cell_dofs(mesh, ku)
    pd = fem.cell_dofs(mesh, kp)
    Lu = np.prod(meshmod.lattice_size(mesh, ku))
    Lp = np.prod(meshmod.lattice_size(mesh, kp))
    cache = {}
    elems = []
    rows, cols, mv, kv = [], [], [], []
    grows, gcols, gx, gy = [], [], [], []
    for c, dv, dp in zip(mesh.cells, vd, pd):
        verts = mesh.vertices[c]
        key = tuple(np.round((verts - verts[0]) / mesh.h).astype(int).ravel())
        if key not in cache:
            cache[key] = fem.taylor_hood_element(ku, kp, verts)
        Mv, Kv, G, To = cache[key]
        elems.append((dv, dp, To))
        rows.append(np.repeat(dv, dv.size))
        cols.append(np.tile(dv, dv.size))
        mv.append(Mv.ravel())
        kv.append(Kv.ravel())
        grows.append(np.repeat(dv, dp.size))
        gcols.append(np.tile(dp, dv.size))
        gx.append(G[0].ravel())
        gy.append(G[1].ravel())
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    M = sp.csr_matrix((np.concatenate(mv), (rows, cols)), shape=(Lu, Lu))
    K = sp.csr_matrix((np.concatenate(kv), (rows, cols)), shape=(Lu, Lu))
    gr, gc = np.concatenate(grows), np.concatenate(gcols)
    Gx = sp.csr_matrix((np.concatenate(gx), (gr, gc)), shape=(Lu, Lp))
    Gy = sp.csr_matrix((np.concatenate(gy), (gr, gc)), shape=(Lu, Lp))
    for A in (M, K, Gx, Gy):
        A.sum_duplicates()
    return M, K, Gx, Gy, elems, Lu, Lp


class NSProblem:
    """Space-time Taylor-Hood x DG(q) discretisation on one mesh level."""

    def __init__(self, mesh, k, q, N, dt, R, bc="lid", lid_speed=1.0):
        if R <= 0:
            raise ValueError("Reynolds number must be > 0")
        self.mesh, self.k, self.ku, self.kp = mesh, k, k + 1, k
        self.q, self.N, self.dt, self.R = int(q), int(N), float(dt), float(R)
        self.tm = dg.TemporalMatrices(q, dt)
        self.Mu, self.Ku, self.Gx, self.Gy, self.elems, self.Lu, self.Lp = _assemble_th(mesh, self.ku, self.kp)
        Lu, Lp = self.Lu, self.Lp
        self.ns = 2 * Lu + Lp
        self.nnode = self.ns  # spatial unknowns (sids): smoother / transfer interface
        self.NT = self.N * (self.q + 1)
        Z = sp.csr_matrix((Lu, Lu))
        self.M2 = sp.bmat([[self.Mu, None, None], [None, self.Mu, None], [None, None, sp.csr_matrix((Lp, Lp))]],
                          format="csr")
        self.K2 = sp.bmat([[self.Ku, None, None], [None, self.Ku, None], [None, None, sp.csr_matrix((Lp, Lp))]],
                          format="csr")
        Gv = sp.bmat([[None, None, self.Gx], [None, None, self.Gy], [self.Gx.T, self.Gy.T, None]], format="csr")
        Gv.resize((self.ns, self.ns))
        self.Gb = Gv.tocsr()  # both off-diagonal blocks (plain transposes, R17)
        del Z
        bnd = meshmod.boundary_nodes(mesh, self.ku)
        self.constrained = np.concatenate([bnd, bnd, np.zeros(Lp, dtype=bool)])
        self.free = ~self.constrained
        self.con_st = np.repeat(self.constrained, self.NT)
        # boundary values (R5): lid (lid_speed, 0) on y = Y except the corners; 0 elsewhere
        xy = meshmod.node_coords(mesh, self.ku)
        X, Y = mesh.nx * mesh.h, mesh.ny * mesh.h
        tol = 1e-12 * max(X, Y)
        g = np.zeros(self.ns)
        if bc == "lid":
            top = (np.abs(xy[:, 1] - Y) < tol) & (np.abs(xy[:, 0]) > tol) & (np.abs(xy[:, 0] - X) > tol)
            g[:Lu][top] = lid_speed
        elif bc != "dirichlet0":
            raise ValueError(bc)
        self.bc_values = g
        self.g_st = np.repeat(g, self.NT)
        self.vel_xy = xy
        self.p_xy = meshmod.node_coords(mesh, self.kp)

    def set_boundary_data(self, G):
        """Time-dependent Dirichlet data (R5, R28): the constrained
        entries of the space-time vector G (solution layout) replace the per-sid
        boundary values; Newton starts from this lift."""
        G = np.asarray(G, dtype=float).reshape(-1)
        if G.size != self.ndof:
            raise ValueError("boundary data must have ndof entries")
        self.g_st = np.where(self.con_st, G, 0.0)

    # ---------------------------------------------------------------- helpers
    @property
    def ndof(self):
        return self.ns * self.NT

    def slab_indices(self, sids, n):
        sids = np.asarray(sids, dtype=np.int64)
        a = np.arange(self.q + 1)
        return ((sids[:, None] * self.N + n) * (self.q + 1) + a[None, :]).ravel()

    def field_view(self, U):
        """(ns, N, q+1) view of a space-time vector."""
        return np.asarray(U).reshape(self.ns, self.N, self.q + 1)

    def velocity_at(self, U, n, c):
        """Nodal velocity (Lu, 2) of slab n, temporal node c."""
        V = self.field_view(U)
        return np.stack([V[:self.Lu, n, c], V[self.Lu:2 * self.Lu, n, c]], axis=1)

    # ------------------------------------------------------------ convection
    def convection(self, w, newton=True):
        """N(w) = O(w) (+ Q(w)) on the velocity sids, as an (ns x ns) sparse matrix."""
        Lu = self.Lu
        rows, cols, vals = [], [], []
        for dv, dp, To in self.elems:
            wl = w[dv]  # (nloc, 2)
            # O: delta_dd' sum_l sum_d2 w[l,d2] To[d2, i, l, j]
            O = np.einsum("ld,dilj->ij", wl, To)
            for d in range(2):
                rows.append(np.repeat(d * Lu + dv, dv.size))
                cols.append(np.tile(d * Lu + dv, dv.size))
                vals.append(O.ravel())
            if newton:
                # Q[(d,i),(d',j)] = sum_l w[l,d] To[d', i, j, l]
                for d in range(2):
                    for d2 in range(2):
                        Q = np.einsum("l,ijl->ij", wl[:, d], To[d2])
                        rows.append(np.repeat(d * Lu + dv, dv.size))
                        cols.append(np.tile(d2 * Lu + dv, dv.size))
                        vals.append(Q.ravel())
        A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                          shape=(self.ns, self.ns))
        A.sum_duplicates()
        return A

    # ----------------------------------------------------- space-time matrices
    def _spacetime(self, blocks):
        """Sum over (row slab, col slab, spatial S, temporal tau) of S (x) tau
        placed in the waveform-major ordering."""
        nq, N = self.q + 1, self.N
        rows, cols, vals = [], [], []
        for nr, nc, S, tau in blocks:
            S = S.tocoo()
            for a in range(nq):
                for b in range(nq):
                    if tau[a, b] == 0.0 or S.nnz == 0:
                        continue
                    rows.append((S.row * N + nr) * nq + a)
                    cols.append((S.col * N + nc) * nq + b)
                    vals.append(S.data * tau[a, b])
        A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                          shape=(self.ndof, self.ndof))
        A.sum_duplicates()
        return A

    def _linear_blocks(self):
        tm = self.tm
        blocks = []
        for n in range(self.N):
            blocks += [(n, n, self.M2, tm.C + tm.E0), (n, n, self.K2, tm.Mt), (n, n, self.Gb, tm.Mt)]
            if n > 0:
                blocks.append((n, n - 1, -self.M2, tm.E1))
        return blocks

    def _identity_rows(self, A):
        keep = sp.diags((~self.con_st).astype(float))
        A = (keep @ A + sp.diags(self.con_st.astype(float))).tocsr()
        A.eliminate_zeros()
        return A

    def jacobian(self, W, newton=True):
        """Newton (or Picard/Oseen) Jacobian at the space-time state W."""
        blocks = self._linear_blocks()
        for n in range(self.N):
            for c in range(self.q + 1):
                Nc = self.convection(self.velocity_at(W, n, c), newton=newton)
                blocks.append((n, n, self.R * Nc, self.tm.T[:, :, c]))
        return self._identity_rows(self._spacetime(blocks))

    def linear_operator(self):
        return self._identity_rows(self._spacetime(self._linear_blocks()))

    def residual(self, U, u0=None):
        """Nonlinear residual F(U) of eq. nsfem (constrained rows U - g)."""
        A = self._spacetime(self._linear_blocks())
        F = A @ U
        Fv = F.reshape(self.ns, self.N, self.q + 1)
        V = self.field_view(U)
        for n in range(self.N):
            for c in range(self.q + 1):
                O = self.convection(self.velocity_at(U, n, c), newton=False)
                for b in range(self.q + 1):
                    ob = O @ V[:, n, b]
                    for a in range(self.q + 1):
                        Fv[:, n, a] += self.R * self.tm.T[a, b, c] * ob
        if u0 is not None:  # slab-0 jump term phi_a(0) M u0 moves to the right-hand side (R7)
            Mu0 = self.M2 @ u0
            Fv[:, 0, :] -= np.outer(Mu0, self.tm.phi0)
        F = Fv.reshape(-1)
        F[self.con_st] = U[self.con_st] - self.g_st[self.con_st]
        return F

    def jacobian_residual_rows(self, rows, x, b, W, newton=True):
        """(b - J(W) x) on the given sids for every (slab, temporal node), evaluated
        row by row from the element integrals (no global space-time matrix): the
        linear rows of M2, K2 + G (eq. nsfem), the jump
        -E1 (x) M2 (R1), and R sum_{b,c} T_abc (N(w_{n,c}) x_{n,b}) with N = O (+ Q)
        (R18) summed over the cells that contain the row's node.  Constrained rows:
        b - x (R5).  Returns an array (len(rows), N, q+1)."""
        nq, N, tm, Lu = self.q + 1, self.N, self.tm, self.Lu
        X, Bv, Wv = self.field_view(x), self.field_view(b), self.field_view(W)
        L2 = (self.K2 + self.Gb).tocsr()
        out = np.zeros((len(rows), N, nq))
        for ir, r in enumerate(rows):
            r = int(r)
            if self.constrained[r]:
                out[ir] = Bv[r] - X[r]
                continue
            mrow, lrow = self.M2.getrow(r), L2.getrow(r)
            Mx = np.einsum("j,jnb->nb", mrow.data, X[mrow.indices]) if mrow.nnz else np.zeros((N, nq))
            Lx = np.einsum("j,jnb->nb", lrow.data, X[lrow.indices]) if lrow.nnz else np.zeros((N, nq))
            acc = Mx @ (tm.C + tm.E0).T + Lx @ tm.Mt.T  # acc[n, a] = sum_b CE_ab Mx[n,b] + Mt_ab Lx[n,b]
            acc[1:, 0] -= Mx[:-1, nq - 1]               # jump: -(E1 M x_{n-1})_a, E1 = e_0 e_q^T (R2)
            if r < 2 * Lu:  # convection rows
                d, i = divmod(r, Lu)
                Nx = np.zeros((N, nq, nq))  # Nx[n, c, b] = (N(w_{n,c}) x_{n,b})_r
                for dv, dp, To in self.elems:
                    loc = np.nonzero(dv == i)[0]
                    if loc.size == 0:
                        continue
                    li = int(loc[0])
                    wl = np.stack([Wv[dv], Wv[Lu + dv]], axis=-1)       # (nloc, N, nq, 2)
                    xl = np.stack([X[dv], X[Lu + dv]], axis=-1)         # (nloc, N, nq, 2)
                    # O: sum_l sum_d2 w[l,d2] To[d2, li, l, j] x_d[j]
                    Ow = np.einsum("lncd,dlj->ncj", wl, To[:, li])     # (N, nq, nloc)
                    Nx += np.einsum("ncj,jnb->ncb", Ow, xl[..., d])
                    if newton:  # Q: sum_l w[l,d] To[d2, li, j, l] x_d2[j]
                        for d2 in range(2):
                            Qw = np.einsum("lnc,jl->ncj", wl[..., d], To[d2, li])
                            Nx += np.einsum("ncj,jnb->ncb", Qw, xl[..., d2])
                acc += self.R * np.einsum("abc,ncb->na", tm.T, Nx)
            out[ir] = Bv[r] - acc
        return out

    def project_pressure(self, U):
        """Remove the mean of the pressure nodal values per (slab, temporal node) (R19)."""
        V = np.array(self.field_view(U), copy=True)
        P = V[2 * self.Lu:]
        V[2 * self.Lu:] = P - P.mean(axis=0, keepdims=True)
        return V.reshape(-1)


# ------------------------------------------------------------------ patches
def vanka_star_patches(prob):
    """Vanka+star patches (Fig. patches right): for every vertex,
    both velocity components on the closure of its star (every velocity node of
    an incident triangle) and the pressure DoFs of the open star (vertex +
    interiors of incident edges / cells).  Constrained DoFs removed, empty
    patches dropped (R8); sids sorted."""
    mesh, ku, kp, Lu = prob.mesh, prob.ku, prob.kp, prob.Lu
    vd = fem.cell_dofs(mesh, ku)
    pd = fem.cell_dofs(mesh, kp)
    pref = fem.reference_nodes(kp)
    vel = [set() for _ in range(mesh.nvert)]
    pre = [set() for _ in range(mesh.nvert)]
    for c, dv, dp in zip(mesh.cells, vd, pd):
        for v in c:
            vel[int(v)].update(int(x) for x in dv)
        for loc, (a, b) in enumerate(pref):
            kind, which = fem.node_entity(kp, a, b)
            owners = [c[which]] if kind == "v" else ([c[which[0]], c[which[1]]] if kind == "e" else list(c))
            for v in owners:
                pre[int(v)].add(int(dp[loc]))
    out, verts = [], []
    for v in range(mesh.nvert):
        sids = [i for i in vel[v] if not prob.constrained[i]] + [Lu + i for i in vel[v] if not prob.constrained[Lu + i]]
        sids += [2 * Lu + j for j in pre[v]]
        if sids:
            out.append(np.array(sorted(sids), dtype=np.int64))
            verts.append(v)
    return out, np.array(verts)


# ------------------------------------------------------------- multigrid
def inject(fine, coarse, U):
    """State on the coarse level by nodal sampling of the fine one (R13; the
    coarse P_k nodes are fine P_k nodes)."""
    Vf = fine.field_view(U)
    Vc = np.zeros((coarse.ns, coarse.N, coarse.q + 1))
    iu = meshmod.node_index_from_coords(fine.mesh, fine.ku, coarse.vel_xy)
    ip = meshmod.node_index_from_coords(fine.mesh, fine.kp, coarse.p_xy)
    Vc[:coarse.Lu] = Vf[iu]
    Vc[coarse.Lu:2 * coarse.Lu] = Vf[fine.Lu + iu]
    Vc[2 * coarse.Lu:] = Vf[2 * fine.Lu + ip]
    return Vc.reshape(-1)


class NSHierarchy:
    """Levels coarse -> fine; operators = Jacobians at the injected state W.
    smoother_kind = "chebyshev": nu_pre / nu_post Chebyshev-accelerated relaxation
    steps (DESIGN.md R-cheb) with lambda re-estimated at every
    linearisation; weight_mode "none" = unweighted additive patches."""

    def __init__(self, nx, ny, h, k, q, N, dt, R, W=None, bc="lid", n_coarse=4, omega_mg=1.0, newton=True,
                 smoother_kind="damped", nu_pre=1, nu_post=1, weight_mode="pou", cheb_steps=50, cheb_seed=7):
        meshes = [Mesh(nx, ny, h)]
        while min(meshes[-1].nx, meshes[-1].ny) > n_coarse:
            m = meshes[-1]
            meshes.append(Mesh(m.nx // 2, m.ny // 2, 2 * m.h))
        meshes = meshes[::-1]
        self.probs = [NSProblem(m, k, q, N, dt, R, bc=bc) for m in meshes]
        self.omega_mg = omega_mg
        self.newton = newton
        self.smoother_kind, self.nu_pre, self.nu_post = smoother_kind, nu_pre, nu_post
        self.weight_mode, self.cheb_steps, self.cheb_seed = weight_mode, cheb_steps, cheb_seed
        self.P0 = [None]
        for l in range(1, len(self.probs)):
            c, f = self.probs[l - 1], self.probs[l]
            Pu = transfer.interpolation(c.mesh, f.mesh, f.ku)
            Pp = transfer.interpolation(c.mesh, f.mesh, f.kp)
            P = sp.block_diag([Pu, Pu, Pp], format="csr")
            self.P0.append(transfer.correction_interpolation(P, f.constrained, c.constrained))
        self.set_state(np.zeros(self.fine.ndof) if W is None else W)

    @property
    def fine(self):
        return self.probs[-1]

    def set_state(self, W):
        """Linearise every level at W (injected to coarse levels) and factor
        the patch blocks (per patch and slab) and the coarse slab blocks."""
        states = [None] * len(self.probs)
        states[-1] = W
        for l in range(len(self.probs) - 1, 0, -1):
            states[l - 1] = inject(self.probs[l], self.probs[l - 1], states[l])
        self.A, self.factors, self.w = [], [], []
        for l, p in enumerate(self.probs):
            A = p.jacobian(states[l], newton=self.newton)
            self.A.append(A)
            if l > 0:
                patches, _ = vanka_star_patches(p)
                self.factors.append(smoother.PatchFactors(p, A, patches))
                self.w.append(smoother.weights(patches, p.ns, self.weight_mode))
            else:
                self.factors.append(None)
                self.w.append(None)
        self.coarse = PinnedCoarse(self.probs[0], self.A[0])
        self.lam = [None] * len(self.probs)
        if self.smoother_kind == "chebyshev":
            for l in range(1, len(self.probs)):
                self.lam[l] = ns_estimate_lambda(self, l)


class PinnedCoarse:
    """Exact coarse solve: block forward substitution over slabs with the full
    slab block; the first pressure DoF of every temporal node is pinned (its
    rows replaced by identity, right-hand side 0) and the result mean-projected
    (R19)."""

    def __init__(self, prob, A):
        self.prob = prob
        sids = np.arange(prob.ns)
        self.I = [prob.slab_indices(sids, n) for n in range(prob.N)]
        nq = prob.q + 1
        pin = [(2 * prob.Lu * nq) + a for a in range(nq)]  # local rows of the first pressure node
        self.pin = pin
        self.lu, self.L = [], [None]
        for n, I in enumerate(self.I):
            D = A[I][:, I].toarray()
            for r in pin:
                D[r, :] = 0.0
                D[r, r] = 1.0
            self.lu.append(sla.lu_factor(D))
            if n > 0:
                Ln = A[I][:, self.I[n - 1]].toarray()
                Ln[pin, :] = 0.0
                self.L.append(Ln)

    def __call__(self, r):
        x = np.zeros_like(r)
        for n, I in enumerate(self.I):
            rhs = r[I].copy()
            if n > 0:
                rhs -= self.L[n] @ x[self.I[n - 1]]
            rhs[self.pin] = 0.0
            x[I] = sla.lu_solve(self.lu[n], rhs)
        return self.prob.project_pressure(x)


def ns_relaxation(H, l, r):
    """B r: one undamped additive Vanka+star sweep from zero, pressure projected (R19)."""
    p = H.probs[l]
    return p.project_pressure(smoother.wr_sweep(p, H.A[l], np.zeros_like(r), r, H.factors[l], 1.0, H.w[l]))


def ns_estimate_lambda(H, l):
    """Largest |Ritz value| of the Arnoldi (CGS2) Hessenberg of B A (DESIGN.md
    R-cheb), start vector = the R6 generator at canonical ids with constrained
    rows 0 (as for heat, multigrid.estimate_lambda)."""
    import wrmg_inputs as wi
    p, A, steps = H.probs[l], H.A[l], H.cheb_steps
    v = wi.uniform_pm1(np.arange(p.ndof, dtype=np.uint64), H.cheb_seed)
    v[p.con_st] = 0.0
    V = [v / np.linalg.norm(v)]
    Hm = np.zeros((steps + 1, steps))
    for j in range(steps):
        w = ns_relaxation(H, l, A @ V[j])
        Vm = np.array(V)
        h = Vm @ w
        w = w - Vm.T @ h
        h2 = Vm @ w
        w = w - Vm.T @ h2
        Hm[:j + 1, j] = h + h2
        Hm[j + 1, j] = np.linalg.norm(w)
        V.append(w / Hm[j + 1, j])
    return float(np.abs(np.linalg.eigvals(Hm[:steps, :steps])).max())


def ns_chebyshev(H, l, u, b, nu):
    """nu Chebyshev steps on [0.25 lam, 1.05 lam], as
    multigrid.chebyshev with the Navier-Stokes relaxation."""
    A, lam = H.A[l], H.lam[l]
    lo, hi = 0.25 * lam, 1.05 * lam
    theta, delta = 0.5 * (hi + lo), 0.5 * (hi - lo)
    sigma = theta / delta
    rho = 1.0 / sigma
    d = ns_relaxation(H, l, b - A @ u) / theta
    u = u + d
    for _ in range(1, nu):
        rn = 1.0 / (2.0 * sigma - rho)
        d = rn * rho * d + (2.0 * rn / delta) * ns_relaxation(H, l, b - A @ u)
        rho = rn
        u = u + d
    return u


def vcycle(H, r, l=None):
    """V(1,1) with the additive Vanka+star waveform smoother; pressure projected
    after every smoother application and on the cycle output (R19).  With
    smoother_kind = "chebyshev": V(nu_pre, nu_post) Chebyshev-accelerated."""
    if l is None:
        l = len(H.probs) - 1
    p = H.probs[l]
    if l == 0:
        return H.coarse(r)
    A = H.A[l]
    cheb = H.smoother_kind == "chebyshev"
    if cheb:
        u = ns_chebyshev(H, l, np.zeros_like(r), r, H.nu_pre)
    else:
        u = smoother.wr_sweep(p, A, np.zeros_like(r), r, H.factors[l], H.omega_mg, H.w[l])
        u = p.project_pressure(u)
    res = r - A @ u
    rc = transfer.restrict(H.P0[l], res, p.NT)
    ec = vcycle(H, H.probs[l - 1].project_pressure(rc), l - 1)
    u = u + transfer.prolong(H.P0[l], ec, p.NT)
    if cheb:
        return ns_chebyshev(H, l, u, r, H.nu_post)
    u = smoother.wr_sweep(p, A, u, r, H.factors[l], H.omega_mg, H.w[l])
    return p.project_pressure(u)


def eisenstat_walker(eta_prev, fn, fn_prev, gamma=1.0, alpha=(1 + 5 ** 0.5) / 2, eta_max=0.9):
    """Choice 2 of Eisenstat & Walker with the safeguard (R22)."""
    eta = gamma * (fn / fn_prev) ** alpha
    if gamma * eta_prev ** alpha > 0.1:
        eta = max(eta, gamma * eta_prev ** alpha)
    return min(eta, eta_max)


def newton(H, rtol=1e-8, maxit=20, eta0=0.3, restart=30, u0=None):
    """Newton-FGMRES-WRMG: full steps from the boundary lift."""
    from . import krylov
    p = H.fine
    U = p.g_st.copy()
    F = p.residual(U, u0)
    f0 = np.linalg.norm(F)
    hist, lin = [f0], []
    eta, fprev = eta0, f0
    for it in range(maxit):
        if np.linalg.norm(F) <= rtol * f0:
            break
        H.set_state(U)
        A = H.A[-1]
        b = -F
        b[p.con_st] = -F[p.con_st]
        b = p.project_pressure(b)
        dx, its, h, st = krylov.fgmres(lambda v: A @ v, lambda r: vcycle(H, r), b, restart=restart,
                                       maxit=200, rtol=eta)
        lin.append(its)
        U = p.project_pressure(U + dx)
        F = p.residual(U, u0)
        fn = np.linalg.norm(F)
        hist.append(fn)
        eta = eisenstat_walker(eta, fn, fprev)
        fprev = fn
    return U, hist, lin


# ------------------------------------------------------- error functional
def triangle_rule(npts):
    """Collapsed (Duffy) Gauss-Legendre rule on the reference triangle
    {xi, eta >= 0, xi + eta <= 1}: xi = u, eta = v (1 - u), weight (1 - u);
    exact for polynomials of degree <= 2 npts - 2.  Returns (points (n, 2), weights)."""
    g, w = np.polynomial.legendre.leggauss(npts)
    g, w = 0.5 * (g + 1.0), 0.5 * w
    U, V = np.meshgrid(g, g, indexing="ij")
    WU, WV = np.meshgrid(w, w, indexing="ij")
    pts = np.stack([U.ravel(), (V * (1.0 - U)).ravel()], axis=1)
    return pts, (WU * WV * (1.0 - U)).ravel()


def velocity_l2_error(prob, U, exact, nspace=6, ntime=None):
    """Space-time L2 norm of the velocity error (Table
    tab:chorin:mg_errors):  ( sum_n int_{I_n} int_Omega |u_h - u|^2 )^(1/2),
    u_h = sum_i sum_a U[(d,i), n, a] v_i(x) phi_a((t - t_n)/dt) on slab n, by the
    collapsed Gauss rule per triangle (nspace^2 points) and Gauss-Legendre in time
    (ntime points, default q + 4).  exact(x, y, t) -> (ux, uy), broadcasting.
    Post-processing for tests; not part of the solver."""
    ku, mesh, N, q, dt = prob.ku, prob.mesh, prob.N, prob.q, prob.dt
    ntime = q + 4 if ntime is None else ntime
    xi, wx = triangle_rule(nspace)
    B = fem.evaluate_basis(ku, xi)                        # (nqp, nloc)
    gt, wt = np.polynomial.legendre.leggauss(ntime)
    gt, wt = 0.5 * (gt + 1.0), 0.5 * wt
    Tb = prob.tm.eval(gt)                                 # (ntime, q+1)
    dofs = fem.cell_dofs(mesh, ku)                        # (ncell, nloc)
    V = prob.field_view(U)
    vx = mesh.vertices[mesh.cells]                        # (ncell, 3, 2)
    J1, J2 = vx[:, 1] - vx[:, 0], vx[:, 2] - vx[:, 0]
    det = np.abs(J1[:, 0] * J2[:, 1] - J1[:, 1] * J2[:, 0])   # (ncell,)
    X = vx[:, None, 0, :] + xi[None, :, 0:1] * J1[:, None, :] + xi[None, :, 1:2] * J2[:, None, :]
    tot = 0.0
    for n in range(N):
        t = (n + gt) * dt
        ex = exact(X[:, :, 0:1], X[:, :, 1:2], t[None, None, :])       # each (ncell, nqp, ntime)
        err = 0.0
        for comp in (0, 1):
            coef = V[comp * prob.Lu + dofs, n, :]                    # (ncell, nloc, q+1)
            uh = np.einsum("ql,cla,ta->cqt", B, coef, Tb)
            err = err + (uh - ex[comp]) ** 2
        tot += dt * np.einsum("c,q,t,cqt->", det, wx, wt, err)
    return float(np.sqrt(tot))
