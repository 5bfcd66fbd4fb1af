#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 300 python tools/prof_ns_factor.py > gpurun_out/nsf_plain.log 2>&1
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:k_ns_factor -c 1 -o /tmp/nsf python tools/prof_ns_factor.py > gpurun_out/nsf_ncu.log 2>&1
ncu -i /tmp/nsf.ncu-rep --page source --csv > gpurun_out/nsf_source.csv 2>/dev/null
ncu -i /tmp/nsf.ncu-rep --page details --csv > gpurun_out/nsf_details.csv 2>/dev/null
ls -la gpurun_out/nsf*
