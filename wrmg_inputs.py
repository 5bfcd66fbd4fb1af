"""Seeded synthetic inputs shared by the oracle and the CUDA path.

Holds none of the method's arithmetic: only the counter-based generator of
DESIGN.md R6 and the canonical-index helpers needed to call it.  Both
``oracle/`` and the tests/bench use it to draw the SAME inputs; the CUDA library
carries its own independent implementation of the same generator
(csrc/kernels_misc.cu, ``wrmg_fill_uniform``), checked equal by tests.

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
