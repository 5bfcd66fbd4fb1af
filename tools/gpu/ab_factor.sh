timeout 900 python -m pytest tests/test_gpu_ns.py tests/test_gpu_ns_windows.py tests/test_gpu_ns_strips.py -x -q > gpurun_out/b_nstest.log 2>&1; echo rc=$? >> gpurun_out/b_nstest.log
timeout 300 python tools/time_ns_factor.py >> gpurun_out/b_time.log 2>&1
timeout 300 python tools/time_ns_factor.py --c4 --slabs 8 >> gpurun_out/b_time.log 2>&1
