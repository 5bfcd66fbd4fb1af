timeout 900 python -m pytest tests/test_gpu_residual_mac.py tests/test_gpu_launchpaths.py -x -q -p no:cacheprovider > gpurun_out/r2_t28.log 2>&1; echo rc=$? >> gpurun_out/r2_t28.log
