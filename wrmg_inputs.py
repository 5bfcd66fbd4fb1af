"""Seeded synthetic inputs shared by the oracle and the CUDA path.

Holds none of the method's arithmetic: only the counter-based generator of
DESIGN.md R6 and the canonical-index helpers needed to call it.  Both
``oracle/`` and the tests/bench use it to draw the SAME inputs; the CUDA library
carries its own independent implementation of the same generator
(csrc/kernels_solve.cu ``k_fill_uniform``, exported as ``wrmg_fill_uniform``), checked equal by tests.

splitmix64 finaliser at canonical id g (uint64, mod 2^64):
    z = g + (seed + 1) * 0x9E3779B97F4A7C15
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
    z = (z ^ (z >> 27)) * 0x94D049BB133111EB
    z ^= z >> 31
    v = 2 * (z >> 11) * 2^-53 - 1          in [-1, 1)
"""
import numpy as np

_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def uniform_pm1(ids, seed=0):
    """U[-1, 1) values at uint64 canonical ids (array-like)."""
    z = np.asarray(ids, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(seed + 1) * _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return 2.0 * (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) - 1.0


def spacetime_field(nnode, N, q, seed=0, node_offset=0):
    """Waveform-major field over nnode spatial nodes: value at canonical id
    ((node_offset + i) * N + n) * (q + 1) + a (R4, R6)."""
    nt = N * (q + 1)
    ids = np.arange(nnode * nt, dtype=np.uint64) + np.uint64(node_offset * nt)
    return uniform_pm1(ids, seed)


def wind_state(nx, ny, h, k, N, q, dt):
    """Linearisation state of config C3 (BASELINE.json configs[2]; R18):
    the nodal values of w = curl psi = (d_y psi, -d_x psi),
    psi = a(t) sin^2(pi x) sin^2(pi y), a(t) = 1 + sin(2 pi t) / 2, at every
    P_{k+1} velocity node and every DG(q) temporal node t = (n + a/q) dt (R2;
    t = n dt for q = 0); pressure 0.  Waveform-major over sids (u_x, u_y, p)."""
    ku, kp = k + 1, k
    Lux, Luy = ku * nx + 1, ku * ny + 1
    Lp = (kp * nx + 1) * (kp * ny + 1)
    I, J = np.meshgrid(np.arange(Lux), np.arange(Luy), indexing="xy")
    x, y = I.ravel() * h / ku, J.ravel() * h / ku
    tau = np.array([0.0]) if q == 0 else np.arange(q + 1) / q
    t = ((np.arange(N)[:, None] + tau[None, :]) * dt).ravel()  # (N (q+1),)
    amp = 1.0 + 0.5 * np.sin(2 * np.pi * t)
    wx = np.pi * np.sin(np.pi * x) ** 2 * np.sin(2 * np.pi * y)
    wy = -np.pi * np.sin(2 * np.pi * x) * np.sin(np.pi * y) ** 2
    out = np.zeros((2 * Lux * Luy + Lp, t.size))
    out[:Lux * Luy] = np.outer(wx, amp)
    out[Lux * Luy:2 * Lux * Luy] = np.outer(wy, amp)
    return out.ravel()


def paper_heat_u0(nx, ny, h, k):
    """Initial state of the paper's heat runs: the nodal values
    of u0(x, y) = sin(pi x) + cos(2 pi y) on the P_k lattice, canonical order."""
    Lx, Ly = k * nx + 1, k * ny + 1
    I, J = np.meshgrid(np.arange(Lx), np.arange(Ly), indexing="xy")
    x, y = I.ravel() * h / k, J.ravel() * h / k
    return np.sin(np.pi * x) + np.cos(2 * np.pi * y)


def chorin_velocity(x, y, t):
    """Exact velocity of the Chorin problem:
    u = (-cos(pi x) sin(pi y), sin(pi x) cos(pi y)) exp(-2 pi^2 t).  Broadcasts."""
    e = np.exp(-2.0 * np.pi ** 2 * t)
    return (-np.cos(np.pi * x) * np.sin(np.pi * y) * e, np.sin(np.pi * x) * np.cos(np.pi * y) * e)


def chorin_pressure(x, y, t, R):
    """Pressure that makes chorin_velocity a solution of u_t - Lap u + R (u.grad)u
    + grad p = 0 (R27 reading: the printed +R pi/4 (...) does not;
    -R/4 (cos 2 pi x + cos 2 pi y) exp(-4 pi^2 t) does).  Reference only."""
    return -0.25 * R * (np.cos(2 * np.pi * x) + np.cos(2 * np.pi * y)) * np.exp(-4.0 * np.pi ** 2 * t)


def _velocity_nodes(nx, ny, h, k):
    ku = k + 1
    Lux, Luy = ku * nx + 1, ku * ny + 1
    I, J = np.meshgrid(np.arange(Lux), np.arange(Luy), indexing="xy")
    return I.ravel() * h / ku, J.ravel() * h / ku, (k * nx + 1) * (k * ny + 1)


def chorin_boundary_data(nx, ny, h, k, N, q, dt):
    """Dirichlet data of the Chorin runs (R28) in the Taylor-Hood
    waveform-major layout (sids u_x, u_y, p): in space the exact velocity at every
    P_{k+1} node; in time, per slab, the degree-q polynomial interpolating it at the
    q+1 Gauss-Legendre points (the slab midpoint for q = 0), stored as its values at
    the DG(q) nodes t = (n + a/q) dt of R2.  Pressure 0.  Only the boundary rows
    are used by the solvers."""
    x, y, Lp = _velocity_nodes(nx, ny, h, k)
    g = 0.5 * (np.polynomial.legendre.leggauss(q + 1)[0] + 1.0)     # interpolation points in [0, 1]
    tau = np.array([0.0]) if q == 0 else np.arange(q + 1) / q       # R2 nodes
    # L[a, j] = Lagrange polynomial of point g_j evaluated at node tau_a
    L = np.ones((q + 1, q + 1))
    for j in range(q + 1):
        for m in range(q + 1):
            if m != j:
                L[:, j] *= (tau - g[m]) / (g[j] - g[m])
    tg = ((np.arange(N)[:, None] + g[None, :]) * dt)                  # (N, q+1)
    ux, uy = chorin_velocity(x[:, None, None], y[:, None, None], tg[None, :, :])
    ux, uy = np.einsum("aj,snj->sna", L, ux), np.einsum("aj,snj->sna", L, uy)
    return np.concatenate([ux.reshape(x.size, -1), uy.reshape(x.size, -1), np.zeros((Lp, N * (q + 1)))]).ravel()


def chorin_u0(nx, ny, h, k):
    """Initial state of the Chorin runs: exact velocity at t = 0 on the P_{k+1}
    nodes, pressure 0 (sid vector)."""
    x, y, Lp = _velocity_nodes(nx, ny, h, k)
    ux, uy = chorin_velocity(x, y, 0.0)
    return np.concatenate([ux, uy, np.zeros(Lp)])
