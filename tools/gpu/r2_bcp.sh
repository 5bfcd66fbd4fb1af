#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_launchpaths.py tests/test_gpu_fullsize.py -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/bcp_t.log
for cfg in "0 0" "1 0" "1 1"; do set -- $cfg
WRMG_BOUNDARY_CP=$1 WRMG_SWEEP_CP=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bcp_$1$2.json 2> gpurun_out/bcp_$1$2.err
done
cat gpurun_out/bcp_t.log
python - <<'P'
import json
for f in ("00","10","11"):
    d=json.loads(open(f"gpurun_out/bcp_{f}.json").read().strip().splitlines()[-1])
    print(f, d["value"], d["ms_per_step"], d["fgmres_iterations"], " ".join(f"{k}:{v['ms']}" for k,v in d["per_kernel"].items() if k.startswith("sweep")))
P
