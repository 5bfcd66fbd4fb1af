#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_launchpaths.py -q -p no:cacheprovider -k symmetric 2>&1 | tail -5 > gpurun_out/cp_t.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cp_b.json 2> gpurun_out/cp_b.err
WRMG_SWEEP_CP=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cp_b0.json 2> gpurun_out/cp_b0.err
cat gpurun_out/cp_t.log
python - <<'P'
import json
for f in ("gpurun_out/cp_b.json","gpurun_out/cp_b0.json"):
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], d["ms_per_step"], d["fgmres_iterations"])
    for k,v in d["per_kernel"].items():
        if k.startswith("sweep"): print("  ",k,v)
P
