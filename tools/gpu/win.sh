timeout 900 python -m pytest tests/test_gpu_ns_windows.py tests/test_gpu_ns.py -x -q > gpurun_out/w_test.log 2>&1; echo rc=$? >> gpurun_out/w_test.log
timeout 1500 python bench.py --config C4 --c4-n 128 --steps 1 --warmup 3 > gpurun_out/w_c4full.json 2> gpurun_out/w_c4full.err
