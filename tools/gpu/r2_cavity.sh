#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python tools/paper_cavity_table.py 2 1 2 > gpurun_out/cav_m2.jsonl 2> gpurun_out/cav_m2.err
timeout 2400 python tools/paper_cavity_table.py 3 2 > gpurun_out/cav_m3.jsonl 2> gpurun_out/cav_m3.err
tail -3 gpurun_out/cav_m2.err gpurun_out/cav_m3.err
cat gpurun_out/cav_m2.jsonl gpurun_out/cav_m3.jsonl
