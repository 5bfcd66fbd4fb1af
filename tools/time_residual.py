"""Times the finest-level residual r = b - A u of C2 (P3 x DG1, 128^2, 128 slabs): 20 launches."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2407_13997_b200 as w  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
c = w.Context(n, n, 1.0 / n, degree=3, q=1, nslabs=128, dt=1.0 / 128, kappa=1.0)
u, b, r = c.empty(), c.empty(), c.empty()
c.fill_uniform(u, 0, 1)
c.fill_uniform(b, 0, 2)
for _ in range(5):
    c.residual(u, b, r)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    c.residual(u, b, r)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
nb = 24.0 * c.layout["ndof"]
print(f"n={n} residual {ms * 1e3:.1f} us  {nb / (ms / 1e3) / 1e9:.0f} GB/s")
