timeout 900 python -m pytest tests/test_gpu_ns_factor_paths.py tests/test_gpu_ns_windows.py -x -q > gpurun_out/g_test.log 2>&1; echo rc=$? >> gpurun_out/g_test.log
python bench.py --config C4 --steps 1 --warmup 3 > gpurun_out/g_c4.json 2> gpurun_out/g_c4.err
