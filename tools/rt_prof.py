"""Phase timers of the register-tiled NS block inversion (WRMG_NS_FACTOR_RT=9): one C3
linearisation, clock64 cycles per block for each phase."""
import ctypes
import os
import sys

os.environ["WRMG_NS_FACTOR_RT"] = "9"
import torch

sys.path.insert(0, ".")
import paper_2407_13997_b200 as w  # noqa: E402
from paper_2407_13997_b200 import _lib  # noqa: E402
import wrmg_inputs as wi  # noqa: E402

n, k, q, N = 64, 1, 1, int(sys.argv[1]) if len(sys.argv) > 1 else 8
c = w.Context(n, n, 1.0 / n, degree=k, q=q, nslabs=N, dt=1.0 / 64, problem="ns", reynolds=100.0, bc="lid",
              omega_mg=0.8)
W = torch.as_tensor(wi.wind_state(n, n, 1.0 / n, k, N, q, 1.0 / 64), device="cuda:0")
arr = (ctypes.c_ulonglong * 16)()
c.linearize(W)
torch.cuda.synchronize()
_lib.lib.wrmg_debug_rt_prof(arr)
c.linearize(W)
torch.cuda.synchronize()
_lib.lib.wrmg_debug_rt_prof(arr)
nb = arr[15]
names = {0: "assembly+norm (warp sum)", 1: "acc: mask+X", 2: "acc: update", 3: "acc: owner start->handover",
         4: "acc: barrier wait", 5: "acc: elimination total", 8: "panel: wait handover", 9: "panel: factor",
         10: "panel: barrier wait", 12: "output (warp sum)"}
print("blocks", nb)
for i, nm in names.items():
    print(f"{nm:30s} {arr[i] / nb:12.0f} cycles/block (summed over the role's warps)")
