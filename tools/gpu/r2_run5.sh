timeout 600 python -m pytest tests/test_gpu_residual_mac.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/r2_t5.log 2>&1; echo rc=$? >> gpurun_out/r2_t5.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b5.json 2> gpurun_out/r2_b5.err
python tools/prof_c2_kernels.py > gpurun_out/r2_prof_plain5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_residual_mac_l1" -s 1 -c 1 -o gpurun_out/r2_ncu5 python tools/prof_c2_kernels.py > gpurun_out/r2_ncu5.log 2>&1
