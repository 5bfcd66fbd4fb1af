timeout 900 python -m pytest tests/test_gpu_ns.py tests/test_gpu_ns_windows.py -x -q > gpurun_out/c4f_test.log 2>&1; echo rc=$? >> gpurun_out/c4f_test.log
timeout 300 python tools/time_ns_factor.py --c4 --slabs 8 > gpurun_out/c4f_time.log 2>&1
