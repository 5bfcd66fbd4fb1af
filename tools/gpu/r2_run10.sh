timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_strips.py -x -q -p no:cacheprovider > gpurun_out/r2_t10.log 2>&1; echo rc=$? >> gpurun_out/r2_t10.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --scatter colour > gpurun_out/r2_b10_colour.json 2> gpurun_out/r2_b10_colour.err
