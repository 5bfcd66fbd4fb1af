"""CPU oracle for the space-time waveform-relaxation multigrid hot path (arXiv 2407.13997).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import anything
from this package.  The product path (``paper_2407_13997_b200``) never imports,
links or executes it, and this package never imports the product path.  The two
share no code; the only shared module is ``wrmg_inputs`` (seeded input
generators, no method arithmetic).

Everything here is plain, slow and written to be checked against the paper by
eye: NumPy/SciPy in float64, explicit sparse matrices, per-(patch, slab) LAPACK
LU factorisations, textbook FGMRES.  Every function cites the PAPER.md passage
(line numbers refer to /root/reference/PAPER.md) or the DESIGN.md reading (R#,
see DESIGN.md "Readings") it follows.

Modules
-------
mesh       structured anti-diagonal triangulation, P_k node lattice, entities
fem        reference P_k element by Vandermonde + exact monomial integration
dg         DG(q) temporal matrices on [0,1]
heat       space-time heat operator (eq. heatfem), RHS, residual
patches    vertex-star patches (Fig. patches left)
smoother   waveform-relaxation additive patch smoother
transfer   P_h by finite-element interpolation, P = I (x) P_h, R = P^T
multigrid  semi-coarsened hierarchy, coarse solve, V-cycle
krylov     FGMRES with CGS2

Parity pins: see tests/test_oracle_*.py.  Functions with no independent pin are
marked "parity unpinned" in their docstring and in DESIGN.md.
"""
