timeout 600 python -m pytest tests/test_gpu_host_api.py tests/test_gpu_guard.py -x -q -p no:cacheprovider > gpurun_out/r2_t32.log 2>&1; echo rc=$? >> gpurun_out/r2_t32.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b32.json 2> gpurun_out/r2_b32.err
