#!/bin/bash
# NS strips parity + heat strips regression (one GPU, loopback transport)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_ns_strips.py -x -q 2>&1 | tail -30 > gpurun_out/nsstrips.log
timeout 900 python -m pytest tests/test_gpu_strips.py -x -q 2>&1 | tail -5 >> gpurun_out/nsstrips.log
cat gpurun_out/nsstrips.log
