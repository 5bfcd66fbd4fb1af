"""Short driver for ncu captures of the Navier-Stokes block inversion (H5): the C3
discretisation (P2-P1 x DG1, 64^2, Re 100, wind state) with 8 slabs, one linearisation."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2407_13997_b200 as w  # noqa: E402
import wrmg_inputs as wi  # noqa: E402

n, k, q, N = 64, 1, 1, 8
c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / 64, problem="ns", reynolds=100.0, bc="lid",
              omega_mg=0.8)
W = torch.as_tensor(wi.wind_state(n, n, 1.0 / n, k, N, q, 1.0 / 64), device="cuda:0")
c.linearize(W)
torch.cuda.synchronize()
print("ok")
