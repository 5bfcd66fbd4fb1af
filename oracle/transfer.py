"""Grid transfers.

"P = I (x) P_h, where I is an identity operator over the temporal mesh and P_h
is the standard finite-element interpolation from grid 2h to grid h ... For
restriction from this grid, we use R = P^T."  DESIGN.md R12: P_h[i, J] is the
coarse basis function J evaluated at fine node i (the lattices are nested).
DESIGN.md R5: for corrections, rows of constrained fine DoFs and columns of
constrained coarse DoFs are zeroed (homogeneous boundary conditions on
corrections; restricted residuals vanish on constrained coarse rows).
"""
import numpy as np
import scipy.sparse as sp

from . import fem
from . import mesh as meshmod


def interpolation(coarse, fine, k, drop=1e-13):
    """Raw P_h: (fine lattice nodes) x (coarse lattice nodes)."""
    fxy = meshmod.node_coords(fine, k)
    nf = fxy.shape[0]
    Lxc, Lyc = meshmod.lattice_size(coarse, k)
    nc = Lxc * Lyc
    cdofs = fem.cell_dofs(coarse, k)
    val = {}
    eps = 1e-10
    for c, d in zip(coarse.cells, cdofs):
        v = coarse.vertices[c]
        Jac = np.column_stack([v[1] - v[0], v[2] - v[0]])
        lo, hi = v.min(axis=0) - 1e-12, v.max(axis=0) + 1e-12
        cand = np.nonzero((fxy[:, 0] >= lo[0]) & (fxy[:, 0] <= hi[0])
                          & (fxy[:, 1] >= lo[1]) & (fxy[:, 1] <= hi[1]))[0]
        xi = np.linalg.solve(Jac, (fxy[cand] - v[0]).T).T
        inside = (xi[:, 0] >= -eps) & (xi[:, 1] >= -eps) & (xi.sum(axis=1) <= 1 + eps)
        cand, xi = cand[inside], xi[inside]
        phi = fem.evaluate_basis(k, xi)  # (ncand, nloc)
        for row, vals in zip(cand, phi):
            if row in val:
                continue
            val[row] = (d, vals)
    rows, cols, data = [], [], []
    for row, (d, vals) in val.items():
        keep = np.abs(vals) > drop
        rows.append(np.full(keep.sum(), row))
        cols.append(d[keep])
        data.append(vals[keep])
    P = sp.csr_matrix((np.concatenate(data), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(nf, nc))
    return P


def correction_interpolation(P, con_fine, con_coarse):
    """P_h with constrained fine rows and constrained coarse columns zeroed."""
    Df = sp.diags((~con_fine).astype(float))
    Dc = sp.diags((~con_coarse).astype(float))
    P0 = (Df @ P @ Dc).tocsr()
    P0.eliminate_zeros()
    return P0


def prolong(P0, e_coarse, NT):
    """(I (x) P_h) e in waveform-major ordering: space outermost, so the
    Kronecker product is P_h (x) I_NT."""
    ec = np.asarray(e_coarse).reshape(P0.shape[1], NT)
    return (P0 @ ec).reshape(-1)


def restrict(P0, r_fine, NT):
    """R = P^T applied to a fine vector."""
    rf = np.asarray(r_fine).reshape(P0.shape[0], NT)
    return (P0.T @ rf).reshape(-1)
