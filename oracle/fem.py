"""Continuous Lagrange P_k elements on triangles, by Vandermonde inversion and
exact monomial integration (R20: exact integration of every
polynomial integrand).

Reference triangle T^ = {(xi, eta): xi, eta >= 0, xi + eta <= 1}.  Nodes are
the equispaced lattice points (a/k, b/k), a + b <= k.  The basis phi_i is the
polynomial of degree k with phi_i(node_j) = delta_ij, obtained by inverting the
Vandermonde matrix of the monomials xi^p eta^s (p + s <= k).  Integrals use
    int_T^ xi^p eta^s = p! s! / (p + s + 2)!.

Physical element with vertices v0, v1, v2:  x = v0 + Jac xi,  Jac = [v1-v0, v2-v0].
    mass       M_ij = |det Jac| int_T^ phi_i phi_j
    stiffness  K_ij = |det Jac| int_T^ (Jac^-T grad phi_i) . (Jac^-T grad phi_j)
These are the spatial bilinear forms (U, psi) and (grad U, grad psi) of
eq. heatfem, with the inner product of eq. inner
(PAPER.md:176-180).
"""
from math import factorial

import numpy as np
import scipy.sparse as sp

from . import mesh as meshmod


def reference_nodes(k):
    """[(a, b)] integer lattice coordinates of the P_k reference nodes."""
    return [(a, b) for b in range(k + 1) for a in range(k + 1 - b)]


def monomials(k):
    return [(p, s) for p in range(k + 1) for s in range(k + 1 - p)]


def mono_integral(p, s):
    """int over the reference triangle of xi^p eta^s."""
    return factorial(p) * factorial(s) / factorial(p + s + 2)


def lagrange_coefficients(k):
    """C[m, i]: phi_i = sum_m C[m, i] * mono_m."""
    nodes = np.array(reference_nodes(k), dtype=float) / k
    mons = monomials(k)
    V = np.array([[x ** p * y ** s for (p, s) in mons] for (x, y) in nodes])
    return np.linalg.inv(V)


def _poly_product_integral(ca, cb, mons_a, mons_b):
    tot = 0.0
    for ia, (pa, sa) in enumerate(mons_a):
        if ca[ia] == 0.0:
            continue
        for ib, (pb, sb) in enumerate(mons_b):
            if cb[ib] == 0.0:
                continue
            tot += ca[ia] * cb[ib] * mono_integral(pa + pb, sa + sb)
    return tot


def _gradient_coeffs(C, mons):
    """Monomial coefficients of d/dxi and d/deta of each basis function
    (expressed again over the same monomial list, degree k)."""
    idx = {m: i for i, m in enumerate(mons)}
    n = C.shape[1]
    Gx = np.zeros_like(C)
    Gy = np.zeros_like(C)
    for m, (p, s) in enumerate(mons):
        if p > 0:
            Gx[idx[(p - 1, s)], :] += p * C[m, :]
        if s > 0:
            Gy[idx[(p, s - 1)], :] += s * C[m, :]
    return Gx, Gy


def reference_matrices(k):
    """Reference mass Mh and the three gradient-product matrices
    S_xx, S_xy, S_yy with S_ab[i, j] = int_T^ d_a phi_i d_b phi_j."""
    mons = monomials(k)
    C = lagrange_coefficients(k)
    Gx, Gy = _gradient_coeffs(C, mons)
    n = C.shape[1]
    Mh = np.zeros((n, n))
    S = {key: np.zeros((n, n)) for key in ("xx", "xy", "yx", "yy")}
    for i in range(n):
        for j in range(n):
            Mh[i, j] = _poly_product_integral(C[:, i], C[:, j], mons, mons)
            S["xx"][i, j] = _poly_product_integral(Gx[:, i], Gx[:, j], mons, mons)
            S["xy"][i, j] = _poly_product_integral(Gx[:, i], Gy[:, j], mons, mons)
            S["yx"][i, j] = _poly_product_integral(Gy[:, i], Gx[:, j], mons, mons)
            S["yy"][i, j] = _poly_product_integral(Gy[:, i], Gy[:, j], mons, mons)
    return Mh, S


def element_matrices(k, verts):
    """Mass and stiffness of the physical triangle with vertices verts (3x2)."""
    Mh, S = reference_matrices(k)
    v0, v1, v2 = np.asarray(verts, dtype=float)
    Jac = np.column_stack([v1 - v0, v2 - v0])
    det = abs(np.linalg.det(Jac))
    Ji = np.linalg.inv(Jac)
    G = Ji @ Ji.T  # grad_x phi = Ji^T grad_xi phi  ->  (grad u . grad v) = g_xi^T (Ji Ji^T) g_xi
    K = det * (G[0, 0] * S["xx"] + G[0, 1] * S["xy"] + G[1, 0] * S["yx"] + G[1, 1] * S["yy"])
    return det * Mh, K


def element_node_coords(k, verts):
    v0, v1, v2 = np.asarray(verts, dtype=float)
    Jac = np.column_stack([v1 - v0, v2 - v0])
    nodes = np.array(reference_nodes(k), dtype=float) / k
    return v0[None, :] + nodes @ Jac.T


def cell_dofs(mesh, k):
    """(ncell, nloc) canonical lattice indices of each cell's local nodes."""
    out = []
    for c in mesh.cells:
        xy = element_node_coords(k, mesh.vertices[c])
        out.append(meshmod.node_index_from_coords(mesh, k, xy))
    return np.array(out, dtype=np.int64)


def assemble(mesh, k):
    """Global spatial mass M and stiffness K (CSR, all lattice nodes)."""
    Lx, Ly = meshmod.lattice_size(mesh, k)
    n = Lx * Ly
    dofs = cell_dofs(mesh, k)
    rows, cols, mv, kv = [], [], [], []
    cache = {}
    for c, d in zip(mesh.cells, dofs):
        verts = mesh.vertices[c]
        key = tuple(np.round((verts - verts[0]) / mesh.h).astype(int).ravel())
        if key not in cache:
            cache[key] = element_matrices(k, verts)
        Me, Ke = cache[key]
        rows.append(np.repeat(d, d.size))
        cols.append(np.tile(d, d.size))
        mv.append(Me.ravel())
        kv.append(Ke.ravel())
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    M = sp.csr_matrix((np.concatenate(mv), (rows, cols)), shape=(n, n))
    K = sp.csr_matrix((np.concatenate(kv), (rows, cols)), shape=(n, n))
    M.sum_duplicates()
    K.sum_duplicates()
    return M, K


def node_entity(k, a, b):
    """Classify reference node (a, b): ('v', i) vertex i, ('e', (i, j)) interior
    of edge (i, j), or ('c', None) cell interior.  Barycentric weights are
    (k - a - b, a, b)/k on (v0, v1, v2)."""
    lam = (k - a - b, a, b)
    nz = [i for i in range(3) if lam[i] != 0]
    if len(nz) == 1:
        return ("v", nz[0])
    if len(nz) == 2:
        return ("e", tuple(nz))
    return ("c", None)


def evaluate_basis(k, xi):
    """Values of all reference basis functions at reference points xi (n, 2)."""
    mons = monomials(k)
    C = lagrange_coefficients(k)
    xi = np.atleast_2d(xi)
    Vm = np.array([[x ** p * y ** s for (p, s) in mons] for (x, y) in xi])
    return Vm @ C


# --------------------------------------------------------------------------
# Mixed-degree integrals for Taylor-Hood (eq. nsfem).
# Polynomials on T^ as dense coefficient arrays c[p, s] of xi^p eta^s.

def basis_polys(k):
    """List of (k+1, k+1) coefficient arrays of the P_k reference basis."""
    C = lagrange_coefficients(k)
    out = []
    for i in range(C.shape[1]):
        c = np.zeros((k + 1, k + 1))
        for m, (p, s) in enumerate(monomials(k)):
            c[p, s] = C[m, i]
        out.append(c)
    return out


def poly_mul(a, b):
    out = np.zeros((a.shape[0] + b.shape[0] - 1, a.shape[1] + b.shape[1] - 1))
    for p in range(a.shape[0]):
        for s in range(a.shape[1]):
            if a[p, s] != 0.0:
                out[p:p + b.shape[0], s:s + b.shape[1]] += a[p, s] * b
    return out


def poly_int(c):
    tot = 0.0
    for p in range(c.shape[0]):
        for s in range(c.shape[1]):
            if c[p, s] != 0.0:
                tot += c[p, s] * mono_integral(p, s)
    return tot


def poly_dxi(c):
    out = np.zeros_like(c)
    out[:-1, :] = c[1:, :] * np.arange(1, c.shape[0])[:, None]
    return out


def poly_deta(c):
    out = np.zeros_like(c)
    out[:, :-1] = c[:, 1:] * np.arange(1, c.shape[1])[None, :]
    return out


def physical_grads(polys, Jac):
    """(d/dx, d/dy) of each reference polynomial for x = v0 + Jac xi."""
    Ji = np.linalg.inv(Jac)
    out = []
    for c in polys:
        dx, dy = poly_dxi(c), poly_deta(c)
        out.append((Ji[0, 0] * dx + Ji[1, 0] * dy, Ji[0, 1] * dx + Ji[1, 1] * dy))
    return out


def taylor_hood_element(ku, kp, verts):
    """Element integrals on the physical triangle (all times |det Jac|):
    Mv[i,j] = int v_i v_j, Kv[i,j] = int grad v_i . grad v_j          (velocity P_ku)
    G[d][i,j] = int chi_j d_d v_i                                      (pressure P_kp)
    To[d][i,l,j] = int v_i v_l d_d v_j                                 (convection)"""
    v0, v1, v2 = np.asarray(verts, dtype=float)
    Jac = np.column_stack([v1 - v0, v2 - v0])
    det = abs(np.linalg.det(Jac))
    vb, pb = basis_polys(ku), basis_polys(kp)
    vg = physical_grads(vb, Jac)
    nu, npn = len(vb), len(pb)
    Mv = np.array([[poly_int(poly_mul(vb[i], vb[j])) for j in range(nu)] for i in range(nu)]) * det
    Kv = np.array([[poly_int(poly_mul(vg[i][0], vg[j][0]) + 0.0) + poly_int(poly_mul(vg[i][1], vg[j][1]))
                    for j in range(nu)] for i in range(nu)]) * det
    G = np.array([[[poly_int(poly_mul(pb[j], vg[i][d])) for j in range(npn)] for i in range(nu)]
                  for d in range(2)]) * det
    To = np.zeros((2, nu, nu, nu))
    for i in range(nu):
        for l in range(nu):
            vl = poly_mul(vb[i], vb[l])
            for j in range(nu):
                for d in range(2):
                    To[d, i, l, j] = poly_int(poly_mul(vl, vg[j][d]))
    return Mv * 1.0, Kv, G, To * det
