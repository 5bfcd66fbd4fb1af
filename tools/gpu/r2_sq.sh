#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_launchpaths.py tests/test_gpu_fullsize.py tests/test_gpu_edge.py -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/sq_t.log
for v in 1 0; do
WRMG_TRANSFER_SQ=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sq_b$v.json 2> gpurun_out/sq_b$v.err
done
cat gpurun_out/sq_t.log
python - <<'P'
import json
for f in ("sq_b1","sq_b0"):
    d=json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    print(f, d["value"], d["ms_per_step"], d["fgmres_iterations"], " ".join(f"{k}:{v['ms']}" for k,v in d["per_kernel"].items() if k.startswith("prolong") or k.startswith("restrict")))
P
