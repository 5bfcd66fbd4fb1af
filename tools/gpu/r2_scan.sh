timeout 300 python tools/time_sweep_kernel.py 128 64 2>&1 | tail -2 > gpurun_out/scan_time.txt
timeout 900 python -m pytest tests/test_gpu_launchpaths.py tests/test_gpu_parity.py -x -q 2>&1 | tail -5 > gpurun_out/scan_tests.txt
cat gpurun_out/scan_time.txt gpurun_out/scan_tests.txt
