timeout 1200 python -m pytest tests/test_gpu_ns.py tests/test_gpu_paper_chorin.py -x -q -p no:cacheprovider > gpurun_out/r2_t21.log 2>&1; echo rc=$? >> gpurun_out/r2_t21.log
timeout 600 python bench.py --config C3 --steps 3 > gpurun_out/r2_c3wp.json 2> gpurun_out/r2_c3wp.err
timeout 900 python bench.py --config C4 --steps 1 --warmup 1 > gpurun_out/r2_c4wp.json 2> gpurun_out/r2_c4wp.err
