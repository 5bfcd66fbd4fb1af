"""Oracle pins P1-P3: closed-form element matrices, stencils,
basis integrals and the DG(q) temporal matrices, none of them derived from the
oracle's own formulas."""
import numpy as np
import pytest

from oracle import dg, fem, heat, mesh


def test_mesh_invariants():
    m = mesh.Mesh(5, 3, 0.2)
    assert m.ncell == 2 * 5 * 3
    assert np.all(m.signed_areas() > 0)  # CCW
    assert abs(m.signed_areas().sum() - 5 * 3 * 0.04) < 1e-14
    # edges: (3 cells + boundary edges) / 2
    nb = 2 * (5 + 3)
    assert m.edges.shape[0] == (3 * m.ncell + nb) // 2
    # diagonal orientation bottom-right -> top-left: cell (0,0) lower triangle
    assert set(map(tuple, m.vertices[m.cells[0]])) == {(0.0, 0.0), (0.2, 0.0), (0.0, 0.2)}


def test_P1_reference_element():
    # closed forms for the linear triangle (right angle at node 0)
    Mh, S = fem.reference_matrices(1)
    assert np.allclose(Mh, np.array([[2, 1, 1], [1, 2, 1], [1, 1, 2]]) / 24.0, atol=1e-15)
    Kh = S["xx"] + S["yy"]
    assert np.allclose(Kh, [[1, -0.5, -0.5], [-0.5, 0.5, 0], [-0.5, 0, 0.5]], atol=1e-15)


@pytest.mark.parametrize("n", [4, 7])
def test_P1_stencils(n):
    """Interior P1 stencils on the anti-diagonal mesh: stiffness 4 / -1 (axis) /
    0 (anti-diagonal, right-angle cotangent); mass h^2/2 / h^2/12 (6 neighbours)."""
    p = heat.unit_square_problem(n, 1, 0, 1, 1.0, build_matrix=False)
    L = n + 1
    h = 1.0 / n
    I, J = 2, 2
    c = J * L + I
    K = p.K.toarray()[c].reshape(L, L)
    M = p.M.toarray()[c].reshape(L, L)
    assert K[J, I] == pytest.approx(4.0, abs=1e-13)
    for dI, dJ in ((1, 0), (-1, 0), (0, 1), (0, -1)):
        assert K[J + dJ, I + dI] == pytest.approx(-1.0, abs=1e-13)
    for dI, dJ in ((1, -1), (-1, 1)):  # neighbours along the cut diagonal
        assert abs(K[J + dJ, I + dI]) < 1e-13
        assert M[J + dJ, I + dI] == pytest.approx(h * h / 12, rel=1e-13)
    assert abs(K[J + 1, I + 1]) < 1e-13 and abs(M[J + 1, I + 1]) < 1e-16
    assert M[J, I] == pytest.approx(h * h / 2, rel=1e-13)
    assert M.sum() == pytest.approx(h * h, rel=1e-13)
    assert abs(K.sum()) < 1e-12


def _ref_integrals(k):
    Mh, _ = fem.reference_matrices(k)
    return Mh.sum(axis=1), fem.reference_nodes(k)


def test_P2_P3_basis_integrals():
    """int_T phi_i: P2 vertex 0, edge |T|/3; P3 vertex |T|/30, edge 3|T|/40,
    interior 9|T|/20 (textbook closed forms; |T^| = 1/2)."""
    T = 0.5
    expect = {2: {"v": 0.0, "e": T / 3}, 3: {"v": T / 30, "e": 3 * T / 40, "c": 9 * T / 20}}
    for k, table in expect.items():
        ints, nodes = _ref_integrals(k)
        for val, (a, b) in zip(ints, nodes):
            kind, _ = fem.node_entity(k, a, b)
            assert val == pytest.approx(table[kind], abs=1e-13), (k, a, b)


@pytest.mark.parametrize("k", [1, 2, 3])
def test_P2_polynomial_consistency(k):
    """K 1 = 0; K I(x) = K I(y) = 0 on interior rows; for k >= 2,
    K I(x^2 + y^2) = -4 M 1 on interior rows (int grad(x^2+y^2).grad phi = -int 4 phi)."""
    p = heat.unit_square_problem(3, k, 0, 1, 1.0, build_matrix=False)
    xy = mesh.node_coords(p.mesh, k)
    inner = ~mesh.boundary_nodes(p.mesh, k)
    one = np.ones(p.nnode)
    assert np.max(np.abs(p.K @ one)) < 1e-12
    assert np.max(np.abs((p.K @ xy[:, 0])[inner])) < 1e-12
    assert np.max(np.abs((p.K @ xy[:, 1])[inner])) < 1e-12
    if k >= 2:
        lhs = p.K @ (xy[:, 0] ** 2 + xy[:, 1] ** 2)
        rhs = -4 * (p.M @ one)
        assert np.max(np.abs((lhs - rhs)[inner])) < 1e-12


def test_P3_temporal_matrices_closed_forms():
    """DG0, DG1 (nodes {0,1}) and DG2 (nodes {0,1/2,1}) against the textbook 1D
    Lagrange mass / advection matrices."""
    dt = 0.3
    t0 = dg.TemporalMatrices(0, dt)
    assert np.allclose(t0.C, 0) and np.allclose(t0.E0, 1) and np.allclose(t0.E1, 1)
    assert np.allclose(t0.Mt, dt)
    t1 = dg.TemporalMatrices(1, dt)
    assert np.allclose(t1.C + t1.E0, [[0.5, 0.5], [-0.5, 0.5]], atol=1e-15)
    assert np.allclose(t1.Mt, dt * np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]]), atol=1e-15)
    assert np.allclose(t1.E1, [[0, 1], [0, 0]])
    t2 = dg.TemporalMatrices(2, dt)
    C2 = np.array([[-1 / 2, 2 / 3, -1 / 6], [-2 / 3, 0, 2 / 3], [1 / 6, -2 / 3, 1 / 2]])
    assert np.allclose(t2.C, C2, atol=1e-14)
    assert np.allclose(t2.Mt, dt / 30 * np.array([[4, 2, -1], [2, 16, 2], [-1, 2, 4]]), atol=1e-14)
    assert np.allclose(t2.E1, np.outer([1, 0, 0], [0, 0, 1]))
    # trilinear T_abc for DG1: dt * int tau^i (1-tau)^j, e.g. T_000 = dt/4, T_001 = dt/12
    assert t1.T[0, 0, 0] == pytest.approx(dt / 4)
    assert t1.T[0, 0, 1] == pytest.approx(dt / 12)
    assert t1.T[1, 1, 1] == pytest.approx(dt / 4)
