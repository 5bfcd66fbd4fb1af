"""Times the finest-level residual r = b - A u of C2 (P3 x DG1, 128^2, 128 slabs): 20 launches."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2407_13997_b200 as w  # noqa: E402

c = w.Context(128, 128, 1.0 / 128, degree=3, q=1, nslabs=128, dt=1.0 / 128, kappa=1.0)
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
print(f"residual {ms * 1e3:.1f} us  {911.0e6 / (ms / 1e3) / 1e9:.0f} GB/s")
