timeout 900 python -m pytest tests/test_gpu_edge.py tests/test_gpu_parity.py tests/test_gpu_ns.py tests/test_gpu_strips.py -x -q > gpurun_out/k_test.log 2>&1; echo rc=$? >> gpurun_out/k_test.log
python bench.py --no-cpu-baseline > gpurun_out/k_c2.json 2> gpurun_out/k_c2.err
