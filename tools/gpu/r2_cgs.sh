#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cgs_b.json 2> gpurun_out/cgs_b.err
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_launchpaths.py tests/test_gpu_ns.py tests/test_gpu_paper_heat.py tests/test_gpu_strips.py tests/test_gpu_ns_strips.py tests/test_gpu_host_api.py -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/cgs_t.log
cat gpurun_out/cgs_t.log
python - <<'P'
import json
d=json.loads(open("gpurun_out/cgs_b.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["fgmres_iterations"], d["e2e"]["value"])
for k,v in list(d["per_kernel"].items())[:6]: print(k,v)
P
