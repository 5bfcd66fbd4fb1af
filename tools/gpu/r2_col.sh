#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_determinism.py -q -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/col_t.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --scatter colour > gpurun_out/col_b1.json 2> gpurun_out/col_b1.err
WRMG_COLOUR_RMW=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --scatter colour > gpurun_out/col_b0.json 2> gpurun_out/col_b0.err
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/col_ba.json 2> gpurun_out/col_ba.err
cat gpurun_out/col_t.log
python - <<'P'
import json
for f in ("col_b1","col_b0","col_ba"):
    d=json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    print(f, d["value"], d["ms_per_step"], d["fgmres_iterations"], " ".join(f"{k}:{v['ms']}" for k,v in d["per_kernel"].items() if k.startswith("sweep")))
P
