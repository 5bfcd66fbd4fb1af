python tools/prof_c2_kernels.py > gpurun_out/r2_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_residual_mac|k_sweep_sym" -s 1 -c 2 -o gpurun_out/r2_ncu1 python tools/prof_c2_kernels.py > gpurun_out/r2_ncu1.log 2>&1
echo done >> gpurun_out/r2_ncu1.log
