python tools/prof_ns_factor.py > gpurun_out/r2_pnf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_ns_factor" -c 1 -o gpurun_out/r2_ncu_nsf python tools/prof_ns_factor.py > gpurun_out/r2_ncu_nsf.log 2>&1
