#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ns.py tests/test_gpu_ns_strips.py -q -p no:cacheprovider 2>&1 | tail -4 > gpurun_out/la_t.log
for la in 1 0; do
WRMG_NS_FACTOR_LA=$la timeout 600 python bench.py --config C3 --steps 2 --warmup 3 > gpurun_out/la_c3_$la.json 2> gpurun_out/la_c3_$la.err
done
WRMG_NS_FACTOR_LA=1 timeout 900 python bench.py --config C4 --steps 2 --warmup 2 > gpurun_out/la_c4_1.json 2> gpurun_out/la_c4_1.err
cat gpurun_out/la_t.log
python - <<'P'
import json
for f in ("la_c3_1","la_c3_0","la_c4_1"):
    try:
        d=json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, round(d["linearize_ms"],1), {k:v for k,v in d["linearize_kernels"].items() if k.startswith("factor")})
    except Exception as e: print(f, e)
P
