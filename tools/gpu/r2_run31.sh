timeout 1200 python -m pytest tests/test_gpu_ns.py tests/test_gpu_paper_chorin.py -x -q -p no:cacheprovider > gpurun_out/r2_t31.log 2>&1; echo rc=$? >> gpurun_out/r2_t31.log
timeout 600 python bench.py --config C3 --steps 1 > gpurun_out/r2_c3w.json 2>&1
