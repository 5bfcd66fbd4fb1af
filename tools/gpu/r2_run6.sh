nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/atomic_probe tools/atomic_probe.cu && /tmp/atomic_probe > gpurun_out/r2_atomic_probe2.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_residual_mac.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/r2_t6.log 2>&1; echo rc=$? >> gpurun_out/r2_t6.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b6.json 2> gpurun_out/r2_b6.err
python tools/prof_c2_kernels.py > gpurun_out/r2_prof_plain6.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_residual_mac" -s 1 -c 1 -o gpurun_out/r2_ncu6 python tools/prof_c2_kernels.py > gpurun_out/r2_ncu6.log 2>&1
