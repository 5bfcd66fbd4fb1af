"""Vertex-star patches (Fig. patches left).

"Vertex-star patches are defined by taking each vertex in the mesh, identifying
all edges and elements incident on the vertex, and then taking the set of DoFs
associated with the vertex itself and those internal to the incident edges and
elements."  DESIGN.md R8: one patch per vertex, boundary vertices included;
constrained (Dirichlet) DoFs are removed and empty patches dropped; DoFs inside a
patch are ordered by canonical index.  Multiplicities mu_i count the patches that
contain DoF i (R11 weights W = 1/mu).
"""
import numpy as np

from . import fem


def vertex_star_patches(mesh, k, constrained):
    """List of int64 arrays (sorted canonical spatial DoFs), one per non-empty
    vertex patch, in vertex order; and the vertex id of each patch."""
    cdofs = fem.cell_dofs(mesh, k)
    ref = fem.reference_nodes(k)
    stars = [set() for _ in range(mesh.nvert)]
    for c, d in zip(mesh.cells, cdofs):
        for loc, (a, b) in enumerate(ref):
            kind, which = fem.node_entity(k, a, b)
            if kind == "v":
                owners = [c[which]]
            elif kind == "e":
                owners = [c[which[0]], c[which[1]]]
            else:
                owners = list(c)
            for v in owners:
                stars[int(v)].add(int(d[loc]))
    patches, verts = [], []
    for v, s in enumerate(stars):
        p = np.array(sorted(i for i in s if not constrained[i]), dtype=np.int64)
        if p.size:
            patches.append(p)
            verts.append(v)
    return patches, np.array(verts, dtype=np.int64)


def multiplicity(patches, nnode):
    mu = np.zeros(nnode, dtype=np.int64)
    for p in patches:
        mu[p] += 1
    return mu
