#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ns_strips.py tests/test_gpu_ns.py -x -q 2>&1 | tail -8 > gpurun_out/nsstrips2.log
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 > gpurun_out/c3.json 2> gpurun_out/c3.err
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 > gpurun_out/c4.json 2> gpurun_out/c4.err
cat gpurun_out/nsstrips2.log; tail -3 gpurun_out/c3.err gpurun_out/c4.err
python - <<'P'
import json
for f in ("gpurun_out/c3.json","gpurun_out/c4.json"):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d["value"], d["ms_per_step"], d.get("linearize_ms"), d["config"]["workload"][:80])
    except Exception as e: print(f, e)
P
