"""Structured triangulation of [0, nx*h] x [0, ny*h] and its P_k node lattice.

PAPER.md:524-525 (sec. numerics): "regular triangulation of the unit square ...
quadrilateral cells in both the x and y directions cut into 2 triangles each
from bottom-right to top-left".  Uniform refinement of such a
mesh is again such a mesh with half the cell size, so every level of the
hierarchy is built directly here (R14: power-of-two sizes).

Every P_k node of the mesh is a point of the (k*nx+1) x (k*ny+1) lattice of
spacing h/k; the canonical spatial index of a node is  J*(k*nx+1) + I
(R4).  The oracle computes node indices from physical coordinates,
so continuity across cells follows from shared coordinates.
"""
import numpy as np


class Mesh:
    """Vertices, CCW triangles and edges of the anti-diagonal lattice mesh."""

    def __init__(self, nx, ny, h):
        self.nx, self.ny, self.h = int(nx), int(ny), float(h)
        I, J = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), indexing="xy")
        self.vertices = np.stack([I.ravel() * h, J.ravel() * h], axis=1)
        cells = []
        vid = lambda i, j: j * (nx + 1) + i
        for j in range(ny):
            for i in range(nx):
                v00, v10, v11, v01 = vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)
                # diagonal from bottom-right (v10) to top-left (v01)
                cells.append((v00, v10, v01))
                cells.append((v10, v11, v01))
        self.cells = np.array(cells, dtype=np.int64)
        edges = set()
        for c in self.cells:
            for a, b in ((0, 1), (1, 2), (0, 2)):
                edges.add(tuple(sorted((int(c[a]), int(c[b])))))
        self.edges = np.array(sorted(edges), dtype=np.int64)

    @property
    def nvert(self):
        return self.vertices.shape[0]

    @property
    def ncell(self):
        return self.cells.shape[0]

    def signed_areas(self):
        v = self.vertices[self.cells]
        d1, d2 = v[:, 1] - v[:, 0], v[:, 2] - v[:, 0]
        return 0.5 * (d1[:, 0] * d2[:, 1] - d1[:, 1] * d2[:, 0])


def unit_square(n):
    """n x n cells on the unit square."""
    return Mesh(n, n, 1.0 / n)


def lattice_size(mesh, k):
    """Number of P_k nodes per direction: (k*nx+1, k*ny+1)."""
    return k * mesh.nx + 1, k * mesh.ny + 1


def node_index_from_coords(mesh, k, xy):
    """Canonical lattice index of P_k nodes at physical coordinates xy (R4)."""
    Lx, _ = lattice_size(mesh, k)
    I = np.rint(np.asarray(xy)[..., 0] * k / mesh.h).astype(np.int64)
    J = np.rint(np.asarray(xy)[..., 1] * k / mesh.h).astype(np.int64)
    return J * Lx + I


def node_coords(mesh, k):
    """Physical coordinates of every lattice node, canonical order."""
    Lx, Ly = lattice_size(mesh, k)
    I, J = np.meshgrid(np.arange(Lx), np.arange(Ly), indexing="xy")
    return np.stack([I.ravel() * mesh.h / k, J.ravel() * mesh.h / k], axis=1)


def boundary_nodes(mesh, k):
    """Boolean mask of lattice nodes on the boundary of the rectangle."""
    xy = node_coords(mesh, k)
    X, Y = mesh.nx * mesh.h, mesh.ny * mesh.h
    tol = 1e-12 * max(X, Y)
    return ((np.abs(xy[:, 0]) < tol) | (np.abs(xy[:, 0] - X) < tol)
            | (np.abs(xy[:, 1]) < tol) | (np.abs(xy[:, 1] - Y) < tol))
