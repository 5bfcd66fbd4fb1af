"""Finest-level smoother device times (per-kernel CUDA events, wrmg_profile) of a
C2-shaped heat level (P3 x DG1, N = 128) at the meshes given (C2's levels: 128 ... 8):
python tools/time_sweep_kernel.py 128 64 32."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2407_13997_b200 as w  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [128]:
    c = w.Context(n, n, 1.0 / n, degree=3, q=1, nslabs=128, dt=1.0 / 128, kappa=1.0)
    u, b = c.zeros(), c.empty()
    c.fill_uniform(b, 0, 2)
    fin = c.layout["nlevels"] - 1
    for _ in range(3):
        c.smooth(u, b, 1, 0.8)
    torch.cuda.synchronize()
    c.profile(True)
    for _ in range(20):
        c.smooth(u, b, 1, 0.8)
    c.sync()
    st = c.kernel_stats()
    c.profile(False)
    print(f"n={n} " + ", ".join(f"{k[0]}@L{k[1]}={v['ms'] / v['launches'] * 1e3:.1f} us x {v['launches'] // 20}"
                                for k, v in st.items() if k[1] == fin), flush=True)
    c.close()
