#!/usr/bin/env python
"""Print the headline numbers and per-kernel table of a bench JSON line."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print({k: d.get(k) for k in ["value", "ms_per_step", "fgmres_iterations", "vcycle_ms", "smoother_sweep_ms",
                             "gpu_launches"]})
print("roofline", {k: d["roofline"][k] for k in ["bound", "achieved", "peak", "frac", "kernel", "share_of_kernel_time"]})
print("clocks", d.get("clocks"), "e2e", round(d["e2e"]["value"] / 1e9, 3), "G")
steps = d["steps"]
for k, v in list(d["per_kernel"].items())[:int(sys.argv[2]) if len(sys.argv) > 2 else 16]:
    print(f"{k:14s} {v['ms'] / steps:8.3f} ms/step {v['ms'] / v['launches'] * 1e3:9.1f} us/launch  "
          f"{v['GBs']} GB/s {v['TFs']} TF/s")
