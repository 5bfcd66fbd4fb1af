"""Upwind DG(q) in time on one slab, mapped to the reference interval [0, 1].

Eq. dgintime summed over slabs I_n = (t_n, t_{n+1}):
    sum_n int_{I_n} (Y_t + L Y) . phi dt + sum_n [[Y_n]] . phi_n^+ = 0,
    [[Y_n]] = Y_n^+ - Y_n^-,  Y_0^- = y_0.
DESIGN.md R1: Y_n^+ is the value at the start of slab n and Y_n^- the value at
the end of slab n-1 (the trace arrows at PAPER.md:97-99 are swapped relative to
the upwind scheme that PAPER.md:120,127 require).
DESIGN.md R2: Lagrange nodal basis on q+1 equispaced nodes including both end
points (q >= 1); DG0 is the constant 1.

With U|_{I_n}(t_n + dt*tau) = sum_b U_{n,b} phi_b(tau) and test phi_a:
    int_{I_n} U_t phi_a dt    = sum_b C_ab U_{n,b},     C_ab = int_0^1 phi_b' phi_a
    phi_a(0) U_n^+            = sum_b E0_ab U_{n,b},    E0_ab = phi_a(0) phi_b(0)
    phi_a(0) U_n^-            = sum_b E1_ab U_{n-1,b},  E1_ab = phi_a(0) phi_b(1)
    int_{I_n} U phi_a dt      = sum_b Mt_ab U_{n,b},    Mt_ab = dt int_0^1 phi_a phi_b
    int_{I_n} w U phi_a dt    = sum_bc T_abc w_c U_b,   T_abc = dt int_0^1 phi_a phi_b phi_c
"""
import numpy as np
from numpy.polynomial import polynomial as P


class TemporalMatrices:
    def __init__(self, q, dt):
        self.q, self.dt = int(q), float(dt)
        nodes = np.array([0.0]) if q == 0 else np.linspace(0.0, 1.0, q + 1)
        self.nodes = nodes
        basis = []
        for a in range(q + 1):
            c = np.array([1.0])
            for b in range(q + 1):
                if b != a:
                    c = P.polymul(c, np.array([-nodes[b], 1.0]) / (nodes[a] - nodes[b]))
            basis.append(c)
        self.basis = basis
        integ = lambda c: float(P.polyval(1.0, P.polyint(c)) - P.polyval(0.0, P.polyint(c)))
        n = q + 1
        self.C = np.array([[integ(P.polymul(P.polyder(basis[b]), basis[a])) for b in range(n)]
                           for a in range(n)])
        v0 = np.array([P.polyval(0.0, c) for c in basis])
        v1 = np.array([P.polyval(1.0, c) for c in basis])
        self.E0 = np.outer(v0, v0)
        self.E1 = np.outer(v0, v1)
        self.Mt = dt * np.array([[integ(P.polymul(basis[a], basis[b])) for b in range(n)]
                                 for a in range(n)])
        self.T = dt * np.array([[[integ(P.polymul(P.polymul(basis[a], basis[b]), basis[c]))
                                  for c in range(n)] for b in range(n)] for a in range(n)])
        self.phi0 = v0
        self.phi1 = v1

    def eval(self, tau):
        """Values of the q+1 basis functions at local times tau."""
        tau = np.atleast_1d(tau)
        return np.array([P.polyval(tau, c) for c in self.basis]).T
