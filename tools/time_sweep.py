"""Times one finest-level smoother sweep of a C2-shaped heat problem (P3 x DG1, N = 128)
at mesh n (C2's levels: 128, 64, 32, 16, 8): 20 sweeps."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2407_13997_b200 as w  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
c = w.Context(n, n, 1.0 / n, degree=3, q=1, nslabs=128, dt=1.0 / 128, kappa=1.0)
u, b = c.zeros(), c.empty()
c.fill_uniform(b, 0, 2)
for _ in range(3):
    c.smooth(u, b, 1, 0.8)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    c.smooth(u, b, 1, 0.8)
e1.record()
torch.cuda.synchronize()
print(f"n={n} sweep {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
