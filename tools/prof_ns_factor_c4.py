"""Short driver for ncu captures of the m = 162 Navier-Stokes block inversion (C4's P3-P2
x DG1 Vanka blocks): 32^2 mesh, 8 slabs, one linearisation at the lid lift."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2407_13997_b200 as w  # noqa: E402

n, k, q, N = 32, 2, 1, 8
c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / 128, problem="ns", reynolds=1000.0, bc="lid",
              omega_mg=0.8)
c.linearize(c.zeros())
torch.cuda.synchronize()
print("ok")
