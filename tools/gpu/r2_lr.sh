#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ns.py tests/test_gpu_ns_strips.py tests/test_gpu_paper_chorin.py -q -p no:cacheprovider 2>&1 | tail -4 > gpurun_out/lr_t.log
for la in 2 1; do
WRMG_NS_FACTOR_LA=$la timeout 600 python bench.py --config C3 --steps 2 --warmup 3 > gpurun_out/lr_c3_$la.json 2> gpurun_out/lr_c3_$la.err
done
timeout 900 python bench.py --config C4 --steps 2 --warmup 2 > gpurun_out/lr_c4.json 2> gpurun_out/lr_c4.err
cat gpurun_out/lr_t.log
python - <<'P'
import json
for f in ("lr_c3_2","lr_c3_1","lr_c4"):
    try:
        d=json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, round(d["linearize_ms"],1), {k:v for k,v in d["linearize_kernels"].items() if k.startswith("factor@L4") or k.startswith("factor@L5")}, d.get("fgmres_iterations"), d.get("fgmres_status_relres"))
    except Exception as e: print(f, e)
P
