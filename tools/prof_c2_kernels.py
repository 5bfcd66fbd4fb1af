"""Short C2-sized driver for ncu captures of the finest-level kernels (not a bench):
residual (H6) and smoother sweep (H7+H8) on the C2 hierarchy, a few calls each."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2407_13997_b200 as w  # noqa: E402

n, k, q, N = 128, 3, 1, 128
c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / N)
u, b, r = c.empty(), c.empty(), c.empty()
c.fill_uniform(u, 0, 1)
c.fill_uniform(b, 0, 2)
for _ in range(3):
    c.residual(u, b, r)
for _ in range(2):
    c.smooth(u, b, 1, 1.0)
x = c.empty()
c.fgmres(b, x, restart=30, maxit=3, rtol=1e-12)
torch.cuda.synchronize()
print("ok")
