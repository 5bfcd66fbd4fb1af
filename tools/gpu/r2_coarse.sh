#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -k "one_level or vcycle" tests/test_gpu_ns.py -q -p no:cacheprovider --durations=5 2>&1 | tail -10 > gpurun_out/co_t.log
timeout 1200 python -m pytest tests/test_gpu_paper_heat.py -q -p no:cacheprovider --durations=5 2>&1 | tail -10 >> gpurun_out/co_t.log
rm -f gpurun_out/chorin_k2.jsonl
WRMG_PAPER_TABLES=1 WRMG_TABLE_OUT=gpurun_out/chorin_k2.jsonl timeout 1800 python -m pytest tests/test_gpu_paper_chorin.py -k "table and 2" -q -p no:cacheprovider -s 2>&1 | tail -12 >> gpurun_out/co_t.log
cat gpurun_out/co_t.log
