set -x
timeout 900 python -m pytest tests/test_gpu_residual_mac.py tests/test_gpu_launchpaths.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q -p no:cacheprovider --durations=8 > gpurun_out/r2_t2.log 2>&1; echo rc=$? >> gpurun_out/r2_t2.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b2.json 2> gpurun_out/r2_b2.err
WRMG_RESIDUAL=tile WRMG_SWEEP_SYM=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b2_old.json 2> gpurun_out/r2_b2_old.err
