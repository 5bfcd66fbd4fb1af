timeout 900 python -m pytest tests/test_gpu_launchpaths.py tests/test_gpu_determinism.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r2_t27.log 2>&1; echo rc=$? >> gpurun_out/r2_t27.log
WRMG_GUARD=1 timeout 900 python tools/guard_check.py > gpurun_out/r2_guard.log 2>&1; echo rc=$? >> gpurun_out/r2_guard.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b27.json 2> gpurun_out/r2_b27.err
